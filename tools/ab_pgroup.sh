#!/bin/bash
# Raster group 16 for the swapped tf32 pair GEMM (RCSG_TC_PAIR_GROUP): cfg2 headline A/B and ncu of step 149.
OUT=${1:-gpurun_out}
for rep in 1 2; do
for G in 1 0; do
  echo "== PAIR_GROUP=$G" >> "$OUT/ab_pgroup.log"
  RCSG_TC_PAIR_GROUP=$G timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-xeb --no-post --scale-configs none --alt-precision none 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg2 tf32', round(d['value'],1), round(r['frac'],3), round(r['launch_ms'],3), d['clocks']['sm_mhz'])" >> "$OUT/ab_pgroup.log" 2>&1
done; done
mkdir -p "$OUT/ncu_top"; timeout -s KILL 500 tools/ncu_top.sh tf32 "$OUT/ncu_top"
