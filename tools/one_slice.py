"""One cfg2 slice bracketed by cudaProfilerStart/Stop (for ncu --profile-from-start off).
Env: PREC (default f16), M (groups, default 64)."""
import sys, os, torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_2406_18889_b200 as pb
prec = os.environ.get("PREC", "f16")
M = int(os.environ.get("M", "64"))
p = pb.Problem(30, 14, "grid(5,6)", 1, list(range(6)), 3 << 30, "low").build()
fixed, _ = pb.build_candidate_set(30, list(range(6)), M, pb.split_next(1, 0xca11d))
acc = torch.zeros(M * 64 * 2, dtype=torch.float64, device='cuda')
for s in range(3):
    p.contract_groups_device(fixed, acc.data_ptr(), precision=prec, configs=None, slices=(s, s + 1))
torch.cuda.synchronize()
torch.cuda.profiler.start()
p.contract_groups_device(fixed, acc.data_ptr(), precision=prec, configs=None, slices=(7, 8))
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
