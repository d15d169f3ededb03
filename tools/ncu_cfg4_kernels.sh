#!/bin/bash
# ncu --set full of selected tcgen05 GEMM launches of one cfg4 slice (launch
# index among gemm_tc_persistent launches, from tools/ncu_slice.sh's join).
# Usage: tools/ncu_cfg4_kernels.sh OUTDIR IDX...
OUT=$1; shift
export CFG=cfg4 PREC=tf32 RCSG_NO_GRAPH=1
for IDX in "$@"; do
  ncu --profile-from-start off --set full --import-source on --clock-control none \
      --kernel-name regex:gemm_tc_persistent --launch-skip "$IDX" --launch-count 1 \
      -o "/tmp/cfg4_k$IDX" -f python tools/one_slice_cfg.py > "$OUT/cfg4_k$IDX.log" 2>&1
  ncu -i "/tmp/cfg4_k$IDX.ncu-rep" --page raw --csv > "$OUT/cfg4_k${IDX}_raw.csv" 2>/dev/null
  ncu -i "/tmp/cfg4_k$IDX.ncu-rep" --page details --csv > "$OUT/cfg4_k${IDX}_details.csv" 2>/dev/null
done
