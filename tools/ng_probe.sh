#!/bin/bash
# Epilogue group count (RCSG_TC_NG) vs per-launch time of one cfg4 / cfg2 tf32 slice (ncu launch lists).
OUT=${1:-gpurun_out}
for NG in auto 1 4; do
  if [ "$NG" = auto ]; then unset RCSG_TC_NG; else export RCSG_TC_NG=$NG; fi
  mkdir -p "$OUT/ng_$NG"
  tools/ncu_slice.sh cfg4 tf32 "$OUT/ng_$NG" > /dev/null 2>&1
  tools/ncu_slice.sh cfg2 tf32 "$OUT/ng_$NG" > /dev/null 2>&1
  rm -f "$OUT/ng_$NG"/launches_*.csv "$OUT/ng_$NG"/order_*.txt
done
