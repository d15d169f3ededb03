"""Long-K tcgen05 GEMM timings (the dominant steps of the scale planner's
cfg3 / cfg4 plans and cfg2's step 149), fp16 and tf32, random operands, plain
row-major output.  Env RCSG_TC_GROUP selects the raster (0 = mixed-radix)."""
import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_18889_b200 import _native
L = _native.testkit()
SHAPES = [("cfg4-1156", 8192, 8192, 131072), ("cfg3-596", 2048, 2048, 524288), ("cfg2-149", 3604, 16384, 4096),
          ("cfg4-1445", 8192, 1024, 131072)]
for prec in (sys.argv[1:] or ["f16", "tf32"]):
    f = L.rcsg_gemm_bench_f16 if prec == "f16" else L.rcsg_gemm_bench_tf32
    peak = 1629.7 if prec == "f16" else 814.85
    for name, m, n, k in SHAPES:
        ms = C.c_double()
        z = (C.c_int8 * 1)()
        rc = f(C.c_int64(m), C.c_int64(n), C.c_int64(k), 0, 0, z, z, 3, C.byref(ms))
        tf = 8.0 * m * n * k / (ms.value * 1e-3) / 1e12
        print(f"{prec:4s} {name:10s} m={m} n={n} k={k} group={os.environ.get('RCSG_TC_GROUP', 'auto')} rc={rc} "
              f"{ms.value:8.3f} ms {tf:7.1f} TF/s frac {tf / peak:.3f}", flush=True)
