#!/bin/bash
# CTA pairs for n = 128 (RCSG_TC_PAIR_MINN=128): cfg4 tf32 rate and amplitude error vs f64.
OUT=${1:-gpurun_out}
for rep in 1 2; do
for N in 128 256; do
  echo "== MINN=$N" >> "$OUT/ab_minn.log"
  RCSG_TC_PAIR_MINN=$N CFG=cfg4 PLAN=plans/cfg4.json TOPN=0 PREC=tf32 SLICES=16 timeout 300 python tools/scale_probe.py 2>/dev/null | tail -1 \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 tf32', round(d['slice_contractions_per_s'],3), round(d['executed_tflops'],1))" >> "$OUT/ab_minn.log" 2>&1
done; done
RCSG_TC_PAIR_MINN=128 CFGS=cfg4 PRECS=tf32 timeout 600 python tools/precision_probe.py >> "$OUT/ab_minn.log" 2>&1
