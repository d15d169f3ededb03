#!/bin/bash
# A/B of RCSG_TC_SLEEPY (producer / MMA threads wait with a suspend-time hint):
# cfg2 headline (tf32, M=1024, 256 slices), cfg4 per-slice (16 slices), long-K GEMMs.
OUT=${1:-gpurun_out}
for S in 0 1 0 1; do
  echo "== SLEEPY=$S" >> "$OUT/sleepy_probe.log"
  RCSG_TC_SLEEPY=$S python bench.py --no-cpu-baseline --no-e2e --no-xeb --no-post --scale-configs none \
      --alt-precision none 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2 tf32', d['value'], d['roofline']['frac'], d['clocks'])" >> "$OUT/sleepy_probe.log" 2>&1
  RCSG_TC_SLEEPY=$S CFG=cfg4 PLAN=plans/cfg4.json TOPN=0 PREC=tf32 SLICES=16 python tools/scale_probe.py 2>/dev/null | tail -1 >> "$OUT/sleepy_probe.log"
done
for S in 0 1; do RCSG_TC_SLEEPY=$S python tools/gemm_big.py tf32 >> "$OUT/sleepy_probe.log" 2>&1; done
