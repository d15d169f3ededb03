"""One tcgen05 GEMM shape (for ncu): env SHAPE=m,n,k PREC=f16|tf32 ITERS."""
import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_18889_b200 import _native
L = _native.testkit()
m, n, k = map(int, os.environ.get("SHAPE", "2048,2048,524288").split(","))
f = L.rcsg_gemm_bench_f16 if os.environ.get("PREC", "f16") == "f16" else L.rcsg_gemm_bench_tf32
ms = C.c_double()
z = (C.c_int8 * 1)()
rc = f(C.c_int64(m), C.c_int64(n), C.c_int64(k), 0, 0, z, z, int(os.environ.get("ITERS", "1")), C.byref(ms))
print(rc, ms.value, 8.0 * m * n * k / ms.value / 1e9, "TF/s")
