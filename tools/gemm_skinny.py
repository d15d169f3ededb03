"""Skinny tcgen05 GEMM timings on cfg2's HBM-bound steps (plan step 619: m = 2^21,
n = 32, k = 16, through its real output map), fp16 and tf32; GB/s = algorithmic
bytes (A + B read once, C written once) / time."""
import sys, ctypes as C
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from paper_2406_18889_b200 import _native
L = _native.testkit()
HBM = 6537.0
def run(prec, name, m, n, k, mp, npos):
    f = L.rcsg_gemm_bench_f16 if prec == "f16" else L.rcsg_gemm_bench_tf32
    eb = 4 if prec == "f16" else 8  # bytes per complex element (planar)
    mb, nb = len(mp), len(npos)
    a = (C.c_int8 * max(mb, 1))(*mp); b = (C.c_int8 * max(nb, 1))(*npos); ms = C.c_double()
    rc = f(C.c_int64(m), C.c_int64(n), C.c_int64(k), mb, nb, a, b, 20, C.byref(ms))
    by = (m * k + n * k + m * n) * eb
    gbs = by / (ms.value * 1e-3) / 1e9
    print(f"{prec:4s} {name:12s} m={m} n={n} k={k} rc={rc} {ms.value*1e3:8.1f} us {gbs:7.0f} GB/s = {gbs/HBM:.2f} of HBM", flush=True)
for prec in ("f16", "tf32"):
    run(prec, "619-real", 1 << 21, 32, 16, [0,1,2,3,4,7,8,9,10,11,13,14,15,16,17,18,19,20,21,24,25], [5,6,12,22,23])
    run(prec, "619-plain", 1 << 21, 32, 16, [], [])
    run(prec, "287-epi2", 1 << 18, 128, 128, list(range(3, 21)), [0, 1, 2, 21, 22, 23, 24])
    run(prec, "317-epi3", 1 << 19, 64, 64, [0, 1, 2, 3] + list(range(10, 25)), list(range(4, 10)))
