#!/bin/bash
# ncu --set full reports (.ncu-rep) of the k = 2^20 post-processing kernels, for local source-level analysis.
OUT=${1:-gpurun_out}
for K in scan_kernel bucket_scatter_kernel bucket_rank_kernel; do
  ncu --profile-from-start off --set full --import-source on --clock-control none \
      --kernel-name regex:$K --launch-count 1 -o "$OUT/rep_$K" -f python tools/post_probe.py > "$OUT/rep_$K.log" 2>&1
done
ls -la $OUT/rep_*.ncu-rep
