"""Per-slice throughput on BASELINE cfg3 (Sycamore-53 layout, m = 12, l = 6): the
repo's planner at a 3 GiB budget, a fixed subset of consecutive slices, M groups.
Env: M (groups, default 64), PREC (default f16), SLICES (timed slices, default 16).
Prints one JSON line; the full run is extrapolated from the per-slice time."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2406_18889_b200 as pb
from paper_2406_18889_b200._native import rcsg_stats

M = int(os.environ.get("M", "64"))
prec = os.environ.get("PREC", "f16")
NS = int(os.environ.get("SLICES", "16"))
t0 = time.time()
p = pb.Problem(53, 12, "sycamore53", 1, list(range(6)), 3 << 30, "low").build()
plan_s = time.time() - t0
fixed, _ = pb.build_candidate_set(53, list(range(6)), M, pb.split_next(1, 0xCA11D))
acc = torch.zeros(M * 64 * 2, dtype=torch.float64, device="cuda")
stream = torch.cuda.ExternalStream(p.stream(prec))
S = 8
for s in range(0, 2 * S, S):  # warm-up: program build, calibration, caches
    p.contract_groups_device(fixed, acc.data_ptr(), precision=prec, configs=None, slices=(s, s + S))
torch.cuda.synchronize()
st = rcsg_stats()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(stream):
    e0.record(stream)
    for s in range(2 * S, 2 * S + NS, S):
        p.contract_groups_device(fixed, acc.data_ptr(), precision=prec, configs=None, slices=(s, s + S),
                                 stats=st, sync=False)
    e1.record(stream)
p.sync(prec)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
rate = NS / (ms / 1e3)
print(json.dumps({
    "workload": "cfg3: sycamore53 m=12 seed=1 l=6 open={0..5}, budget 3*2^30 B",
    "plan_s": round(plan_s, 1), "sliced": len(p.plan["sliced"]), "n_slices": p.n_slices,
    "flops_per_slice_per_group": p.plan["flops_per_slice"], "groups": M, "precision": prec,
    "timed_slices": NS, "ms": ms, "slice_contractions_per_s": rate,
    "executed_tflops": st.executed_flops / (ms / 1e3) / 1e12,
    "reference_equivalent_tflops": p.plan["flops_per_slice"] * M * rate / 1e12,
    "full_run_extrapolated_s": p.n_slices / rate,
    "amps_finite": bool(torch.isfinite(acc).all().item())}))
