#!/bin/bash
# A/B of the pair-GEMM raster rule and the epilogue group count on the cfg2 headline
# (tf32, bench main measurement) and cfg4 per-slice rate, interleaved, same box.
OUT=${1:-gpurun_out}
run() {
  echo "== $1" >> "$OUT/ab_probe.log"
  env $1 python bench.py --no-cpu-baseline --no-e2e --no-xeb --no-post --scale-configs none --alt-precision none 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg2 tf32', round(d['value'],1), round(r['frac'],3), round(r['launch_ms'],3), d['clocks']['sm_mhz'])" >> "$OUT/ab_probe.log" 2>&1
  env $1 CFG=cfg4 PLAN=plans/cfg4.json TOPN=0 PREC=tf32 SLICES=16 python tools/scale_probe.py 2>/dev/null | tail -1 \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 tf32', round(d['slice_contractions_per_s'],3), round(d['executed_tflops'],1))" >> "$OUT/ab_probe.log" 2>&1
}
for rep in 1 2; do
  run "RCSG_TC_PAIR_GROUP=1 RCSG_TC_NG_WIDE=1"
  run "RCSG_TC_PAIR_GROUP=0 RCSG_TC_NG_WIDE=1"
  run "RCSG_TC_PAIR_GROUP=1 RCSG_TC_NG_WIDE=2"
  run "RCSG_TC_PAIR_GROUP=0 RCSG_TC_NG_WIDE=2"
done
