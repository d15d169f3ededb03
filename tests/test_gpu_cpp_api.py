"""The C++ drop-in API on the GPU (tests/cpp/api_gpu.cpp): the program cache
makes the reference's per-group contract_group loop cost about one batched
call, and contract(..., workers) over the device context is bit-identical for
1 and 2 GPUs (the reference's worker-count invariance, test_contraction.cpp:84-93)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2406_18889_b200", "_native")

pytestmark = pytest.mark.gpu


def test_cpp_cache_and_device_context(tmp_path):
    import torch
    n_gpus = torch.cuda.device_count()
    exe = tmp_path / "api_gpu"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "api_gpu.cpp"), "-L", LIB, "-lpaper_2406_18889_b200",
                    f"-Wl,-rpath,{LIB}", "-o", str(exe)], check=True, capture_output=True, timeout=300)
    out = subprocess.run([str(exe), str(min(n_gpus, 2))], check=True, capture_output=True, text=True,
                         timeout=600).stdout
    print(out)
    lines = {" ".join(l.split()[:2]): l.split() for l in out.splitlines()}
    cache = lines["cache compile_ms"]
    compile_ms, batch_ms, loop_ms, worst = float(cache[2]), float(cache[4]), float(cache[6]), float(cache[8])
    assert worst < 1e-12
    # the 64 single-group calls reuse the cached program: no per-call compilation
    assert loop_ms < 64 * compile_ms / 4, (compile_ms, batch_ms, loop_ms)
    m1 = lines["multi slices"]
    assert float(m1[-1]) < 1e-2  # tf32, blocked vs unblocked summation order
    if n_gpus >= 2:
        m2 = lines["multi devices2"]
        assert m2[3] == "1", out
        assert float(m2[-1]) < 1e-2
