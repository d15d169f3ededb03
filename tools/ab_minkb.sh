#!/bin/bash
# A/B of the shortest K that takes CTA-pair tiles (RCSG_TC_PAIR_MINKB, k-blocks of 128 B).
OUT=${1:-gpurun_out}
run() {
  echo "== $1" >> "$OUT/ab_minkb.log"
  env $1 python bench.py --no-cpu-baseline --no-e2e --no-xeb --no-post --scale-configs none --alt-precision none 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg2 tf32', round(d['value'],1), round(r['frac'],3), round(r['launch_ms'],3), d['clocks']['sm_mhz'])" >> "$OUT/ab_minkb.log" 2>&1
  env $1 python bench.py --no-cpu-baseline --no-e2e --no-xeb --no-post --scale-configs none --alt-precision none --precision f16 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg2 f16', round(d['value'],1), round(r['frac'],3), round(r['launch_ms'],3), d['clocks']['sm_mhz'])" >> "$OUT/ab_minkb.log" 2>&1
  env $1 CFG=cfg4 PLAN=plans/cfg4.json TOPN=0 PREC=tf32,f16 SLICES=16 python tools/scale_probe.py 2>/dev/null | tail -2 \
    | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print('cfg4', d['precision'], round(d['slice_contractions_per_s'],3), round(d['executed_tflops'],1))" >> "$OUT/ab_minkb.log" 2>&1
}
for rep in 1 2; do
  run "RCSG_TC_PAIR_MINKB=32"
  run "RCSG_TC_PAIR_MINKB=8"
done
