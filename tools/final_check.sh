#!/bin/bash
# full GPU tests, TMA-store A/B (cfg2 / cfg4 tf32), default bench, smoke
OUT=${1:-gpurun_out}
timeout -s KILL 1100 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo rc=$? >> "$OUT/pytest_gpu.log"
for B in 1 0 1 0; do
  echo "== BLK=$B" >> "$OUT/ab_blk_final.log"
  RCSG_TC_BLK=$B CFG=cfg4 PLAN=plans/cfg4.json TOPN=0 PREC=tf32 SLICES=16 timeout 300 python tools/scale_probe.py 2>/dev/null | tail -1 \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 tf32', round(d['slice_contractions_per_s'],3), round(d['executed_tflops'],1))" >> "$OUT/ab_blk_final.log" 2>&1
done
timeout -s KILL 1300 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo rc=$? >> "$OUT/bench.err"
python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo rc=$? >> "$OUT/smoke.log"
