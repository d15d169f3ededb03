"""The C++ drop-in API (include/rcs_b200.hpp) compiles and links like a
reference-side caller, and its host results equal the reference library's
(same plan, same candidate prefixes).  CPU only: device calls raise
DeviceError without a GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2406_18889_b200", "_native")


def test_cpp_drop_in_compiles_links_and_matches_reference(tmp_path, ref):
    exe = tmp_path / "drop_in"
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "cpp",
           "drop_in.cpp"), "-L", LIB, "-lpaper_2406_18889_b200", f"-Wl,-rpath,{LIB}", "-o", str(exe)]
    subprocess.run(cmd, check=True, capture_output=True, timeout=300)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True, timeout=300).stdout.split("\n")
    steps, sliced, fps = out[0].split()[1], out[0].split()[3], out[0].split()[5]
    r = ref.RefProblem(30, 14, "grid(5,6)", 1, list(range(6)), 3 << 30, "low").build()
    assert int(steps) == len(r.plan["steps"])  # one row per contraction step
    assert int(sliced) == len(r.plan["sliced"])
    assert float(fps) == float(r.plan["flops_per_slice"])
    fixed, dup = ref.candidates(30, list(range(6)), 64, ref.split_next(1, 0xCA11D))
    g0, g63 = out[1].split()[1], out[1].split()[3]
    assert int(g0) == int(fixed[0]) and int(g63) == int(fixed[63])
    assert out[2] == "qsvd 144 3 1"  # 16-byte header + 8 x 16 bytes, round trip exact
    assert out[3].startswith("device")
