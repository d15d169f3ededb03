"""The C-ABI library loads on a CPU host and exports every symbol include/rcsg.h
declares, with struct layouts that match the header (checked by compiling a
probe against the header).  No device calls here."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import pytest

from paper_2406_18889_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rcsg.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(rcsg_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    names = declared_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    for n in _native.RCSH_SYMBOLS:
        assert hasattr(lib, n), n


def test_ctypes_structs_match_header():
    probe = r"""
#include <stddef.h>
#include <stdio.h>
#include "rcsg.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(rcsg_network_desc), sizeof(rcsg_plan_desc), sizeof(rcsg_stats),
         sizeof(rcsg_candidates), offsetof(rcsg_stats, device_ms), offsetof(rcsg_stats, gemm_tc_launches),
         sizeof(rcsg_post_stats), offsetof(rcsg_post_stats, xeb_topk));
  return 0;
}
"""
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "p.c")
        open(src, "w").write(probe)
        exe = os.path.join(d, "p")
        subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), src, "-o", exe], check=True)
        got = list(map(int, subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()))
    want = [C.sizeof(_native.rcsg_network_desc), C.sizeof(_native.rcsg_plan_desc), C.sizeof(_native.rcsg_stats),
            C.sizeof(_native.rcsg_candidates), _native.rcsg_stats.device_ms.offset,
            _native.rcsg_stats.gemm_tc_launches.offset, C.sizeof(_native.rcsg_post_stats),
            _native.rcsg_post_stats.xeb_topk.offset]
    assert got == want


def test_status_codes_match_reference_taxonomy():
    # include/rcs/errors.hpp:9-25: ConfigError 2, NumericFault 3, CapacityError 4
    import paper_2406_18889_b200 as pb
    assert (pb.ConfigError.exit_code, pb.NumericFault.exit_code, pb.CapacityError.exit_code) == (2, 3, 4)
    assert (_native.RCSG_ERR_CONFIG, _native.RCSG_ERR_NUMERIC, _native.RCSG_ERR_CAPACITY) == (2, 3, 4)


def test_cpu_host_rejects_device_calls_loudly():
    """On a host without a GPU the device path fails with DeviceError; it never
    falls back to a CPU computation."""
    import paper_2406_18889_b200 as pb
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    p = pb.Problem(6, 4, "line", 1, [0, 1], 1 << 30, "low").build()
    with pytest.raises(pb.DeviceError):
        p.contract_groups([0], configs=None)
