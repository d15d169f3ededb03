"""fp16 tcgen05 GEMM timings on cfg2 shapes and output maps (rcsg_gemm_bench_f16)."""
import sys, ctypes as C
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from paper_2406_18889_b200 import _native
L = _native.testkit()
f = L.rcsg_gemm_bench_f16
def run(name, m, n, k, mp, npos):
    mb, nb = len(mp), len(npos)
    a = (C.c_int8 * max(mb, 1))(*mp); b = (C.c_int8 * max(nb, 1))(*npos); ms = C.c_double()
    rc = f(C.c_int64(m), C.c_int64(n), C.c_int64(k), mb, nb, a, b, 10, C.byref(ms))
    tiles = (m // 128) * max(1, n // 64)
    print(f"{name:12s} m={m} n={n} k={k} rc={rc} {ms.value*1e3:8.1f} us  {ms.value*1e3/(tiles/148):6.2f} us/tile-round", flush=True)
run("619-real", 1 << 21, 32, 16, [0,1,2,3,4,7,8,9,10,11,13,14,15,16,17,18,19,20,21,24,25], [5,6,12,22,23])
run("619-plain", 1 << 21, 32, 16, [], [])
run("n64k64", 1 << 21, 64, 64, [], [])
run("n64k16", 1 << 21, 64, 16, [], [])
