#!/bin/bash
# 3xtf32 GEMM error vs the fp32 SIMT kernel against the K chunk per split (RCSG_TC_MAX_KB):
# is the remaining error the tensor-core accumulation chain?
OUT=${1:-gpurun_out}
for KB in 100000 256 64 16; do
  echo "== max_kb=$KB" >> "$OUT/split_acc.log"
  RCSG_TC_MAX_KB=$KB python - >> "$OUT/split_acc.log" 2>&1 <<'PY'
import ctypes as C, sys, os
sys.path.insert(0, os.getcwd())
from paper_2406_18889_b200 import _native
L = _native.testkit()
for m, n, k in ((4096, 1024, 8192), (1 << 14, 64, 32768), (4096, 256, 512)):
    z = (C.c_int8 * 1)()
    for name in ("3xtf32", "tf32"):
        f = getattr(L, "rcsg_gemm_check_" + name)
        rel = C.c_double()
        rc = f(C.c_int64(m), C.c_int64(n), C.c_int64(k), 0, 0, z, z, C.byref(rel))
        print(name, m, n, k, rc, rel.value)
PY
done
