"""Tensor-core complex GEMM (tcgen05, every epilogue kind and K-tile width)
against the SIMT kernel of the same storage type on random operands through
explicit output maps, for fp16, bf16 and fp32 (kind::tf32) storage.
rel = ||TC - SIMT|| / ||SIMT||: for 2-byte storage both round the same
fp32-accumulated values, so the bound is a few ulps (2e-3 fp16, 1.6e-2 bf16);
tf32 truncates the fp32 operands to 10 mantissa bits (5e-3); 3xtf32 (hi + lo
operand halves, three products per real product) is fp32-grade (2e-5)."""
import ctypes as C

import pytest

from paper_2406_18889_b200 import _native

pytestmark = pytest.mark.gpu

R19 = [0, 1, 2, 3, 6, 7, 8, 9, 11, 12, 15, 16, 17, 18, 19, 20, 21, 22, 23]  # row run of 4 (epi 3)
CASES = [
    ("plain-k64", 1 << 15, 64, 64, [], []),
    ("plain-k512", 4096, 256, 512, [], []),
    ("row-run", 1 << 19, 64, 64, R19, [4, 5, 10, 13, 14, 24]),
    ("col-run3-rows-follow", 1 << 14, 128, 128, list(range(3, 17)), [0, 1, 2, 17, 18, 19, 20]),
    ("col-run7", 1 << 10, 1 << 14, 256, [7, 8, 9, 10, 11, 12, 13, 21, 22, 23], list(range(7)) + list(range(14, 21))),
    ("mixed-low-bits", 1 << 12, 128, 64, [1, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13], [0, 2, 14, 15, 16, 17, 18]),
    ("narrow-k16", 1 << 16, 32, 16, [0, 1, 2, 3, 4, 7, 8, 9, 10, 11, 13, 14, 15, 16, 17, 18], [5, 6, 12, 19, 20]),
    ("narrow-k32-n128", 1 << 13, 128, 32, [], []),
    ("narrow-n8", 1 << 12, 8, 64, [], []),
    ("narrow-k8-n32", 1 << 15, 32, 8, [], []),
    ("col-run2", 1 << 13, 64, 128, list(range(2, 15)), [0, 1, 15, 16, 17, 18]),
    # 8 m n k >= 2.7e11, k >= 512, n >= 64: the 3M path (T1 = Ar Br, T2 = Ai Bi, T3 = (Ar+Ai)(Br+Bi))
    ("3m-n1024", 4096, 1024, 8192, [], []),
    ("3m-n64-scatter", 1 << 14, 64, 32768, [7, 8, 9, 10, 11, 12, 13] + list(range(0, 7)), list(range(14, 20))),
    # 4-byte outputs with contiguous 16 x 16 blocks (columns at bits 0-3, rows at 4-7): TMA stores
    ("blk16", 1 << 12, 1 << 10, 64, [4, 5, 6, 7] + list(range(14, 22)), [0, 1, 2, 3] + list(range(8, 14))),
    ("blk16-mtail", 4000, 1 << 10, 128, [4, 5, 6, 7] + list(range(14, 22)), [0, 1, 2, 3] + list(range(8, 14))),
    ("blk16-rows", 1 << 12, 1 << 10, 64, [0, 1, 2, 3] + list(range(8, 16)), [4, 5, 6, 7] + list(range(16, 22))),
    ("blk-cols-5d", 1 << 12, 1 << 10, 64, [5, 9, 11, 13] + list(range(14, 22)), [0, 1, 2, 3, 4, 6, 7, 8, 10, 12]),
    # 2-byte outputs: 32-element runs (five column / row bits at output bit 0)
    ("blk2-cols-2d", 1 << 12, 1 << 10, 64, [5, 6, 7, 8] + list(range(14, 22)), [0, 1, 2, 3, 4] + list(range(9, 14))),
    ("blk2-rows-5d", 1 << 12, 1 << 10, 128, [0, 1, 2, 3, 4] + list(range(9, 16)), [5, 7, 8, 16, 6, 17, 18, 19, 20, 21]),
    # CTA-pair tiles (cta_group::2; pair1 = 256 x 128, pair2 = 256 x 256): plain, scatter
    # output, an M tail that leaves the peer CTA without rows, and split K
    ("pair1-plain", 1024, 512, 4096, [], []),
    ("pair2-plain", 1024, 512, 4096, [], []),
    ("pair1-scatter", 1 << 12, 256, 2048, [7, 8, 9, 10, 11, 12, 13, 0, 1, 2, 3, 4], [5, 6] + list(range(14, 20))),
    ("pair2-scatter", 1 << 12, 256, 2048, [7, 8, 9, 10, 11, 12, 13, 0, 1, 2, 3, 4], [5, 6] + list(range(14, 20))),
    ("pair1-mtail", 1000, 768, 2048, [], []),
    ("pair2-mtail", 1000, 768, 2048, [], []),
    ("pair1-splitk", 512, 256, 65536, [], []),
    # m = 3604 (901 row blocks of 4) pads to 3840 on 256-row pairs: computed as the swapped GEMM
    ("pair1-swap", 3604, 512, 2048, [3, 7], [0, 1, 2, 4, 5, 6, 8, 9, 10]),
    ("pair2-splitk", 512, 256, 65536, [], []),
]


@pytest.mark.parametrize("dtype,tol", [("f16", 2e-3), ("bf16", 1.6e-2), ("tf32", 5e-3), ("3xtf32", 2e-5)])
@pytest.mark.parametrize("name,m,n,k,mp,npos", CASES, ids=[c[0] for c in CASES])
def test_tc_gemm_matches_simt(name, m, n, k, mp, npos, dtype, tol, monkeypatch):
    if name.startswith("3m"):
        monkeypatch.setenv("RCSG_TC_3M", "1")  # the opt-in 3M kernel
    if name.startswith("pair"):
        monkeypatch.setenv("RCSG_TC_PAIR", name[4])
    if name.startswith("blk2"):
        monkeypatch.setenv("RCSG_TC_BLK2", "1")  # the opt-in 2-byte TMA-store epilogue
    lib = _native.testkit()
    check = {"f16": lib.rcsg_gemm_check_f16, "bf16": lib.rcsg_gemm_check_bf16, "tf32": lib.rcsg_gemm_check_tf32,
             "3xtf32": lib.rcsg_gemm_check_3xtf32}[dtype]
    a = (C.c_int8 * max(len(mp), 1))(*mp)
    b = (C.c_int8 * max(len(npos), 1))(*npos)
    if dtype == "3xtf32":
        # the tensor cores' fp32 accumulation over a long K chain adds ~3e-9 per k-block of error
        # on top of the split (measured: 1.8e-6 at K = 512, 2.9e-5 at 8192, 5.7e-5 at 32768;
        # 4e-6 at 8192 when every split covers 256 K: profiles/r02/split_acc.log)
        tol = tol * max(1.0, k / 4096)
    rel = C.c_double()
    rc = check(C.c_int64(m), C.c_int64(n), C.c_int64(k), len(mp), len(npos), a, b, C.byref(rel))
    assert rc == 0
    assert rel.value < tol, rel.value
