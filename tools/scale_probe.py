"""Per-slice throughput of the scale planner's plans on BASELINE cfg3-5
(Sycamore-53 m=12 / m=20, Zuchongzhi-60 m=24; l = 6), M groups.
Env: CFG (cfg3|cfg4|cfg5), M, PREC, SLICES (timed), BUDGET_LOG2, TRIALS, PLAN (plan file).
Prints one JSON line per precision."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2406_18889_b200 as pb
from paper_2406_18889_b200._native import rcsg_stats

CFGS = {"cfg3": (53, 12, "sycamore53"), "cfg4": (53, 20, "sycamore53"), "cfg5": (60, 24, "zuchongzhi60")}
cfg = os.environ.get("CFG", "cfg3")
n, m, topo = CFGS[cfg]
M = int(os.environ.get("M", "64"))
NS = int(os.environ.get("SLICES", "16"))
blog = int(os.environ.get("BUDGET_LOG2", "36"))
t0 = time.time()
if os.environ.get("PLAN"):  # a plan file (plans/<cfg>.json) instead of planning here
    p = pb.Problem(n, m, topo, 1, list(range(6)), 1 << blog, "low").build(plan_json=open(os.environ["PLAN"]).read())
else:
    p = pb.Problem(n, m, topo, 1, list(range(6)), 1 << blog, "low").build(planner="scale", n_groups=M,
                                                                         trials=int(os.environ.get("TRIALS", "1024")))
plan_s = time.time() - t0
print(json.dumps({"cfg": cfg, "plan_s": plan_s, "report": p.plan_report, "sliced": len(p.plan["sliced"]),
                  "flops_per_slice_plan": p.plan["flops_per_slice"]}), flush=True)
fixed, _ = pb.build_candidate_set(n, list(range(6)), M, pb.split_next(1, 0xCA11D))
for prec in os.environ.get("PREC", "f16,tf32").split(","):
    acc = torch.zeros(M * 64 * 2, dtype=torch.float64, device="cuda")
    stream = torch.cuda.ExternalStream(p.stream(prec))
    S = min(8, NS)
    tw = time.time()
    for s in range(0, S, S):  # warm-up: program build, reassociation, calibration, caches
        p.contract_groups_device(fixed, acc.data_ptr(), precision=prec, configs=None, slices=(s, s + S))
    torch.cuda.synchronize()
    warm_s = time.time() - tw
    st = rcsg_stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for s in range(S, S + NS, S):
            p.contract_groups_device(fixed, acc.data_ptr(), precision=prec, configs=None, slices=(s, s + S),
                                     stats=st, sync=False)
        e1.record(stream)
    p.sync(prec)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    p.set_profile(True)
    pst = rcsg_stats()
    os.environ["RCSG_PROFILE_STEPS"] = os.environ.get("TOPN", "6")
    p.contract_groups_device(fixed, acc.data_ptr(), precision=prec, configs=None, slices=(0, 1), stats=pst)
    os.environ.pop("RCSG_PROFILE_STEPS")
    p.set_profile(False)
    rate = NS / (ms / 1e3)
    print(json.dumps({"cfg": cfg, "precision": prec, "groups": M, "timed_slices": NS, "ms": ms, "warm_s": warm_s,
                      "slice_contractions_per_s": rate, "executed_tflops": st.executed_flops / (ms / 1e3) / 1e12,
                      "arena_gib": st.arena_bytes / 2**30, "launches": st.kernel_launches,
                      "top": {"step": pst.top_step, "ms": pst.top_ms, "tflops": pst.top_flops / (pst.top_ms * 1e-3) / 1e12 if pst.top_ms else None},
                      "gemm_tc_share": pst.gemm_tc_ms / pst.device_ms if pst.device_ms else None,
                      "full_run_extrapolated_s": p.n_slices / rate,
                      "amps_finite": bool(torch.isfinite(acc).all().item())}), flush=True)
    del acc
    p.release()
