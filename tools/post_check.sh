#!/bin/bash
# post-processing: GPU tests, device-time probe, warm launch list (cache-control none)
OUT=${1:-gpurun_out}
timeout -s KILL 400 python -m pytest tests/test_gpu_postproc.py tests/test_gpu_sampling.py tests/test_gpu_acceptance.py -x -q > "$OUT/t_post.log" 2>&1; echo rc=$? >> "$OUT/t_post.log"
timeout -s KILL 200 python tools/post_timing.py > "$OUT/post_timing.log" 2>&1
timeout -s KILL 300 ncu --profile-from-start off --cache-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file "$OUT/post_launches_warm.csv" python tools/post_probe.py > "$OUT/post_probe.log" 2>&1
