#!/bin/bash
# ncu --set full of the post-processing kernels (tools/post_probe.py calls):
# the bucket rank pass and the fused direct-sampling pass.  Usage: tools/ncu_post_kernels.sh OUTDIR
OUT=${1:-gpurun_out}
for K in bucket_rank_kernel direct_scan_kernel bucket_scatter_kernel sample_hist_kernel; do
  ncu --profile-from-start off --set full --import-source on --clock-control none \
      --kernel-name regex:$K --launch-count 1 -o "/tmp/post_$K" -f python tools/post_probe.py > "$OUT/post_$K.log" 2>&1
  ncu -i "/tmp/post_$K.ncu-rep" --page details --csv > "$OUT/post_${K}_details.csv" 2>/dev/null
  ncu -i "/tmp/post_$K.ncu-rep" --page source --csv > "$OUT/post_${K}_source.csv" 2>/dev/null
done
