"""One slice of a BASELINE config bracketed by cudaProfilerStart/Stop (for ncu
--profile-from-start off), after warm-up slices.  Env: CFG (cfg2 | cfg3 | cfg4:
cfg3/4 use plans/<cfg>.json), PREC (default tf32), M (groups; default 1024 for
cfg2, 64 otherwise), ORDER=1: instead, one profiled slice printing every
launch in issue order ([rcsg-order] lines on stderr) - run with RCSG_NO_GRAPH=1
under ncu so that the launch order is the same."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2406_18889_b200 as pb
from paper_2406_18889_b200._native import rcsg_stats

cfg = os.environ.get("CFG", "cfg2")
prec = os.environ.get("PREC", "tf32")
if cfg == "cfg2":
    M = int(os.environ.get("M", "1024"))
    p = pb.Problem(30, 14, "grid(5,6)", 1, list(range(6)), 3 << 30, "low").build()
    n = 30
else:
    M = int(os.environ.get("M", "64"))
    n, m, topo = {"cfg3": (53, 12, "sycamore53"), "cfg4": (53, 20, "sycamore53")}[cfg]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = pb.Problem(n, m, topo, 1, list(range(6)), 1 << 36, "low").build(
        plan_json=open(os.path.join(root, "plans", cfg + ".json")).read())
fixed, _ = pb.build_candidate_set(n, list(range(6)), M, pb.split_next(1, 0xca11d))
acc = torch.zeros(M * 64 * 2, dtype=torch.float64, device="cuda")
for s in range(2):
    p.contract_groups_device(fixed, acc.data_ptr(), precision=prec, configs=None, slices=(s, s + 1))
torch.cuda.synchronize()
if os.environ.get("ORDER"):
    os.environ["RCSG_PROFILE_ORDER"] = "1"
    p.set_profile(True)
    p.contract_groups_device(fixed, acc.data_ptr(), precision=prec, configs=None, slices=(2, 3), stats=rcsg_stats())
    p.set_profile(False)
else:
    torch.cuda.profiler.start()
    p.contract_groups_device(fixed, acc.data_ptr(), precision=prec, configs=None, slices=(2, 3))
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
torch.cuda.synchronize()
print("ok")
