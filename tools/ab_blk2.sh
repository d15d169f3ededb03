#!/bin/bash
# 2-byte TMA-store epilogue: GEMM tests, A/B on cfg2 / cfg4 fp16, contraction tests.
OUT=${1:-gpurun_out}
timeout -s KILL 400 python -m pytest tests/test_gpu_gemm.py -q > "$OUT/t_blk2.log" 2>&1; echo rc=$? >> "$OUT/t_blk2.log"
timeout -s KILL 600 python -m pytest tests/test_gpu_contract.py -x -q -k "f16 or bf16 or headline" > "$OUT/t_blk2_contract.log" 2>&1; echo rc=$? >> "$OUT/t_blk2_contract.log"
for rep in 1 2; do
for B in 1 0; do
  echo "== BLK=$B" >> "$OUT/ab_blk2.log"
  RCSG_TC_BLK=$B timeout 300 python bench.py --precision f16 --no-cpu-baseline --no-e2e --no-xeb --no-post --scale-configs none --alt-precision none 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg2 f16', round(d['value'],1), round(r['frac'],3), d['clocks']['sm_mhz'])" >> "$OUT/ab_blk2.log" 2>&1
  RCSG_TC_BLK=$B CFG=cfg4 PLAN=plans/cfg4.json TOPN=0 PREC=f16 SLICES=16 timeout 300 python tools/scale_probe.py 2>/dev/null | tail -1 \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 f16', round(d['slice_contractions_per_s'],3), round(d['executed_tflops'],1))" >> "$OUT/ab_blk2.log" 2>&1
done; done
