#!/bin/bash
# per-plane TMA-store maps: GEMM tests, cfg4 slice amplitudes vs RCSG_TC_BLK_PLANES=0 (bitwise), A/B rate
OUT=${1:-gpurun_out}
timeout -s KILL 300 python -m pytest tests/test_gpu_gemm.py -x -q > "$OUT/t_planes.log" 2>&1; echo rc=$? >> "$OUT/t_planes.log"
RCSG_TC_BLK_PLANES=0 timeout 300 python tools/cmp_env.py /tmp/p0.npy > "$OUT/cmp_planes.log" 2>&1
timeout 300 python tools/cmp_env.py /tmp/p1.npy /tmp/p0.npy >> "$OUT/cmp_planes.log" 2>&1
for B in 1 0 1 0; do
  echo "== PLANES=$B" >> "$OUT/ab_planes.log"
  RCSG_TC_BLK_PLANES=$B CFG=cfg4 PLAN=plans/cfg4.json TOPN=0 PREC=tf32 SLICES=16 timeout 300 python tools/scale_probe.py 2>/dev/null | tail -1 \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 tf32', round(d['slice_contractions_per_s'],3), round(d['executed_tflops'],1))" >> "$OUT/ab_planes.log" 2>&1
done
