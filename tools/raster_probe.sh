#!/bin/bash
# Tile-raster group size vs time and DRAM bytes for the dominant cfg2 GEMM
# shape (and the cfg4 long-K one): RCSG_TC_GROUP = 0 (plain) / 4 / 8 / 16.
OUT=${1:-gpurun_out}
for PREC in tf32 f16; do
for SHAPE in 3604,16384,4096 8192,8192,131072; do
for G in 0 4 8 16; do
  echo "== $PREC $SHAPE group=$G" >> "$OUT/raster_probe.log"
  RCSG_TC_GROUP=$G SHAPE=$SHAPE PREC=$PREC ITERS=5 python tools/gemm_one.py >> "$OUT/raster_probe.log" 2>&1
  RCSG_TC_GROUP=$G SHAPE=$SHAPE PREC=$PREC ITERS=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --kernel-name regex:gemm_tc_persistent --launch-count 1 --csv python tools/gemm_one.py 2>/dev/null \
      | grep -E "dram__|gpu__time" | awk -F'","' '{print $(NF-2), $NF}' >> "$OUT/raster_probe.log"
done; done; done
