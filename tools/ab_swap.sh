#!/bin/bash
# A/B of the swapped CTA-pair GEMM (RCSG_TC_SWAP) on the cfg2 headline (tf32) and the GEMM shape.
OUT=${1:-gpurun_out}
timeout -s KILL 300 python -m pytest tests/test_gpu_gemm.py -q -k "pair" > "$OUT/t_pair.log" 2>&1; echo rc=$? >> "$OUT/t_pair.log"
for rep in 1 2; do
for S in 1 0; do
  echo "== SWAP=$S" >> "$OUT/ab_swap.log"
  RCSG_TC_SWAP=$S python bench.py --no-cpu-baseline --no-e2e --no-xeb --no-post --scale-configs none --alt-precision none 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg2 tf32', round(d['value'],1), round(r['frac'],3), round(r['launch_ms'],3), d['clocks']['sm_mhz'])" >> "$OUT/ab_swap.log" 2>&1
done; done
