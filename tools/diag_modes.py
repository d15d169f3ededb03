"""Diagnostics: per-launch profile of one cfg2 call (8 slices, M=1024) per
precision (RCSG_PROFILE_STEPS prints the costliest launches), and the wall time
of consecutive host-buffer contract_groups calls."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2406_18889_b200 as pb
from paper_2406_18889_b200._native import rcsg_stats

M = int(os.environ.get("M", "1024"))
p = pb.Problem(30, 14, "grid(5,6)", 1, list(range(6)), 3 << 30, "low").build()
fixed, _ = pb.build_candidate_set(30, list(range(6)), M, pb.split_next(1, 0xCA11D))
acc = torch.zeros(M * 64 * 2, dtype=torch.float64, device="cuda")
for prec in sys.argv[1:] or ["tf32", "f16"]:
    for s in range(0, 24, 8):
        p.contract_groups_device(fixed, acc.data_ptr(), precision=prec, configs=None, slices=(s, s + 8))
    torch.cuda.synchronize()
    for rep in range(2):
        p.set_profile(True)
        st = rcsg_stats()
        os.environ["RCSG_PROFILE_STEPS"] = "12"
        print(f"== {prec} profiled call {rep}", flush=True)
        p.contract_groups_device(fixed, acc.data_ptr(), precision=prec, configs=None, slices=(32, 40), stats=st)
        p.set_profile(False)
        print(f"   device_ms {st.device_ms:.3f} gemm_tc_ms {st.gemm_tc_ms:.3f} top step {st.top_step} "
              f"top_ms {st.top_ms:.3f} avg {st.top_ms_sum / max(st.top_launches, 1):.3f}", flush=True)
    os.environ.pop("RCSG_PROFILE_STEPS")
    ts = []
    for i in range(6):
        t0 = time.perf_counter()
        out = p.contract_groups(fixed, precision=prec, configs=None, slices=(8 * i, 8 * i + 8))
        ts.append(time.perf_counter() - t0)
    print(f"   host-buffer calls (8 slices) ms: {[round(t * 1e3, 2) for t in ts]}", flush=True)
    st = rcsg_stats()
    t0 = time.perf_counter()
    p.contract_groups_device(fixed, acc.data_ptr(), precision=prec, configs=None, slices=(64, 72), stats=st)
    print(f"   device-buffer sync call ms {1e3 * (time.perf_counter() - t0):.2f} device_ms {st.device_ms:.2f}", flush=True)
