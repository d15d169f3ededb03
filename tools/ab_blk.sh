#!/bin/bash
# TMA-store epilogue (RCSG_TC_BLK): GEMM / contraction tests, A/B on cfg2 and cfg4 (tf32), cfg4 slice launch list.
OUT=${1:-gpurun_out}
timeout -s KILL 400 python -m pytest tests/test_gpu_gemm.py -q > "$OUT/t_blk.log" 2>&1; echo rc=$? >> "$OUT/t_blk.log"
timeout -s KILL 600 python -m pytest tests/test_gpu_contract.py -x -q -k "tf32 or headline" > "$OUT/t_blk_contract.log" 2>&1; echo rc=$? >> "$OUT/t_blk_contract.log"
for rep in 1 2; do
for B in 1 0; do
  echo "== BLK=$B" >> "$OUT/ab_blk.log"
  RCSG_TC_BLK=$B timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-xeb --no-post --scale-configs none --alt-precision none 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg2 tf32', round(d['value'],1), round(r['frac'],3), round(r['launch_ms'],3), d['clocks']['sm_mhz'])" >> "$OUT/ab_blk.log" 2>&1
  RCSG_TC_BLK=$B CFG=cfg4 PLAN=plans/cfg4.json TOPN=0 PREC=tf32 SLICES=16 timeout 300 python tools/scale_probe.py 2>/dev/null | tail -1 \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 tf32', round(d['slice_contractions_per_s'],3), round(d['executed_tflops'],1))" >> "$OUT/ab_blk.log" 2>&1
done; done
mkdir -p "$OUT/blk"; timeout -s KILL 600 tools/ncu_slice.sh cfg4 tf32 "$OUT/blk"; rm -f "$OUT"/blk/launches_* "$OUT"/blk/order_*
