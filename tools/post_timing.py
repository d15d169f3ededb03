"""Device time of rcsg_postprocess at M = 2^20 groups, l = 6, repeated calls:
prints every call's device_ms per mode (top-k 2^20, 2^15, direct, both)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2406_18889_b200 as pb

M, l, n = 1 << 20, 6, 30
g = torch.Generator(device="cuda").manual_seed(1)
amps = torch.randn((M << l) * 2, dtype=torch.float64, device="cuda", generator=g) * 2.0 ** -15
fixed = np.random.default_rng(1).integers(0, 1 << (n - l), size=M, dtype=np.uint64)
op = list(range(6))
for k, d in ((1 << 20, None), (1 << 15, None), (0, 7), (1 << 20, 7)):
    ms, wall = [], []
    for _ in range(12):
        t = time.perf_counter()
        _, _, st = pb.api.postprocess_device_amps(n, op, fixed, amps.data_ptr(), k, direct_seed=d)
        wall.append((time.perf_counter() - t) * 1e3)
        ms.append(st["device_ms"])
    print(f"k={k} direct={d}: device_ms " + " ".join(f"{x:.3f}" for x in ms) +
          f" | wall_ms median {np.median(wall):.2f}", flush=True)
