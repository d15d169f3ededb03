"""fp16 tcgen05 GEMM timings on cfg2 shapes and output maps (rcsg_gemm_bench_f16)."""
import sys, ctypes as C
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from paper_2406_18889_b200 import _native
L = _native.testkit()
f = L.rcsg_gemm_bench_f16
def run(name, m, n, k, mp, npos):
    mb, nb = len(mp), len(npos)
    a = (C.c_int8 * max(mb, 1))(*mp); b = (C.c_int8 * max(nb, 1))(*npos)
    ms = C.c_double()
    rc = f(C.c_int64(m), C.c_int64(n), C.c_int64(k), mb, nb, a, b, 20, C.byref(ms))
    fl = 8.0 * m * n * k
    by = (m * k + n * k + m * n) * 4
    print(f"{name:10s} m={m} n={n} k={k} rc={rc} {ms.value*1e3:8.1f} us  {fl/ms.value/1e9:7.1f} TF/s  {by/ms.value/1e6:7.1f} GB/s", flush=True)
run("317-epi3", 1 << 19, 64, 64, [0, 1, 2, 3] + list(range(10, 25)), list(range(4, 10)))
run("317-plain", 1 << 19, 64, 64, [], [])
run("287-epi2", 1 << 18, 128, 128, list(range(3, 21)), [0, 1, 2, 21, 22, 23, 24])
run("287-plain", 1 << 18, 128, 128, [], [])
run("618-plain", 1 << 14, 1 << 11, 1 << 9, [], [])
run("148-plain", 504, 16384, 2048, [], [])
#run("big", 8192, 8192, 4096, [], [])
run("618-real", 1 << 14, 1 << 11, 1 << 9, [0, 1, 2, 6, 8, 9, 12, 13, 15, 17, 19, 20, 21, 24], [3, 4, 5, 7, 10, 11, 14, 16, 18, 22, 23])
run("148-real", 504, 16384, 2048, [7, 8, 9], list(range(0, 7)) + list(range(10, 17)))
run("619-real", 1 << 21, 32, 16, [0, 1, 2, 3, 4, 7, 8, 9, 10, 11, 13, 14, 15, 16, 17, 18, 19, 20, 21, 24, 25], [5, 6, 12, 22, 23])
