#!/bin/bash
# Per-launch DRAM bytes of one slice: the executor's launch order (profiled run)
# and an ncu launch list with gpu__time_duration + dram read/write bytes of the
# same slice (RCSG_NO_GRAPH=1: single stream, issue order), joined by
# tools/join_slice.py.  Usage: tools/ncu_slice.sh CFG PREC OUTDIR
set -u
CFG=${1:-cfg2}; PREC=${2:-tf32}; OUT=${3:-gpurun_out}
mkdir -p "$OUT"
export CFG PREC RCSG_NO_GRAPH=1
ORDER=1 python tools/one_slice_cfg.py 2> "$OUT/order_${CFG}_${PREC}.txt" > /dev/null
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file "$OUT/launches_${CFG}_${PREC}.csv" python tools/one_slice_cfg.py \
    > "$OUT/ncu_slice_${CFG}_${PREC}.log" 2>&1
python tools/join_slice.py "$OUT/order_${CFG}_${PREC}.txt" "$OUT/launches_${CFG}_${PREC}.csv" \
    > "$OUT/slice_${CFG}_${PREC}.txt"
