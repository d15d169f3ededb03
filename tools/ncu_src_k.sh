#!/bin/bash
# Source-level (CUDA line) ncu profile of one tcgen05 GEMM launch of a cfg4 slice.
# Usage: tools/ncu_src_k.sh OUTDIR IDX
OUT=$1; IDX=$2
export CFG=cfg4 PREC=tf32 RCSG_NO_GRAPH=1
ncu --profile-from-start off --set full --import-source on --clock-control none \
    --kernel-name regex:gemm_tc_persistent --launch-skip "$IDX" --launch-count 1 \
    -o "/tmp/src_k$IDX" -f python tools/one_slice_cfg.py > "$OUT/src_k$IDX.log" 2>&1
ncu -i "/tmp/src_k$IDX.ncu-rep" --page source --csv --print-source cuda > "$OUT/src_k${IDX}_cuda.csv" 2>>"$OUT/src_k$IDX.log"
ncu -i "/tmp/src_k$IDX.ncu-rep" --page details --csv > "$OUT/src_k${IDX}_details.csv" 2>/dev/null
