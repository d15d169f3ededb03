timeout -s KILL 400 python -m pytest tests/test_gpu_postproc.py tests/test_gpu_sampling.py tests/test_gpu_acceptance.py -x -q > gpurun_out/t_post.log 2>&1; echo rc=$? >> gpurun_out/t_post.log
RCSG_TOPK_BUCKETS=0 timeout -s KILL 200 python tools/post_timing.py > gpurun_out/post_timing_radix.log 2>&1
RCSG_TOPK_BUCKETS=1 timeout -s KILL 200 python tools/post_timing.py > gpurun_out/post_timing_buckets.log 2>&1
RCSG_TOPK_BUCKETS=1 timeout -s KILL 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/post_launches.csv python tools/post_probe.py > gpurun_out/post_probe.log 2>&1
