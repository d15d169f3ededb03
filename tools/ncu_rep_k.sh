#!/bin/bash
# ncu --set full report (.ncu-rep, one launch) of a cfg4 tcgen05 GEMM launch, kept for local analysis.
# Usage: tools/ncu_rep_k.sh OUTDIR IDX
OUT=$1; IDX=$2
export CFG=cfg4 PREC=tf32 RCSG_NO_GRAPH=1
ncu --profile-from-start off --set full --import-source on --clock-control none \
    --kernel-name regex:gemm_tc_persistent --launch-skip "$IDX" --launch-count 1 \
    -o "$OUT/rep_k$IDX" -f python tools/one_slice_cfg.py > "$OUT/rep_k$IDX.log" 2>&1
ls -la "$OUT"/rep_k$IDX.ncu-rep >> "$OUT/rep_k$IDX.log"
