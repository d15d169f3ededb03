"""Fused post-processing (rcsg_postprocess, postproc.cu): the threshold-select
top-k, the direct samples drawn in the same streaming pass and the device XEB
must equal the reference sampler (sampling.cpp:62-145) on identical inputs."""
import os

import numpy as np
import pytest

import paper_2406_18889_b200 as pb
from oracle import port

pytestmark = pytest.mark.gpu


def device_amps(M, l, seed, quantize=None):
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    a = torch.randn(M << l, 2, dtype=torch.float64, device="cuda", generator=g) * 2.0**-12
    if quantize:
        a = torch.round(a * quantize) / quantize  # many exactly equal probabilities
    a = a.contiguous()
    h = a.cpu().numpy()
    probs = (h[:, 0] * h[:, 0] + h[:, 1] * h[:, 1]).reshape(M, 1 << l)  # std::norm rounding
    return a, probs


@pytest.mark.parametrize("k", [1, 100, 4096, 65536])
@pytest.mark.parametrize("path", ["auto", "1", "2", "radix", "buckets"])
def test_topk_threshold_select_matches_reference(k, path, monkeypatch):
    """path 1: threshold select, 2: full sort; radix / buckets: threshold
    select ordered by the radix sort + tie pass or by the bucket ranks
    (RCSG_TOPK_BUCKETS=0 / 1)."""
    n, oq, M, l = 30, [0, 1, 2, 3, 4, 5], 4096, 6
    if path in ("radix", "buckets"):
        monkeypatch.setenv("RCSG_TOPK_BUCKETS", "0" if path == "radix" else "1")
    elif path != "auto":
        monkeypatch.setenv("RCSG_TOPK_PATH", path)
    fixed, _ = pb.build_candidate_set(n, oq, M, 1234)
    a, probs = device_amps(M, l, k)
    top, _, st = pb.api.postprocess_device_amps(n, oq, fixed, a.data_ptr(), k)
    want = port.top_k(n, oq, fixed, probs, k)
    assert np.array_equal(top, want)
    if path == "1" or (path == "auto" and 4 * k <= M << l):
        assert st["fast_path"] == 1 and st["candidates_kept"] >= k
    # the sorted prefix really is (prob desc, lexkey asc)
    assert np.array_equal(pb.api.top_k_from_device_amps(n, oq, fixed, a.data_ptr(), k), want)


@pytest.mark.parametrize("order", ["radix", "buckets"])
@pytest.mark.parametrize("quant", [2.0**14, 2.0**11])
def test_topk_ties_short_and_long_runs(quant, order, monkeypatch):
    """Quantised amplitudes give runs of equal probabilities: short runs are
    reordered in place, runs above 256 entries fall back to the full sort."""
    monkeypatch.setenv("RCSG_TOPK_BUCKETS", "0" if order == "radix" else "1")
    n, oq, M, l = 24, [2, 5, 7], 8192, 3
    fixed, _ = pb.build_candidate_set(n, oq, M, 99)
    a, probs = device_amps(M, l, 7, quantize=quant)
    for k in (10, 1000, 5000):
        top, _, st = pb.api.postprocess_device_amps(n, oq, fixed, a.data_ptr(), k)
        assert np.array_equal(top, port.top_k(n, oq, fixed, probs, k)), (quant, k, st)


def test_direct_samples_from_the_fused_pass():
    n, oq, M, l = 30, [0, 1, 2, 3, 4, 5], 2048, 6
    fixed, _ = pb.build_candidate_set(n, oq, M, 5)
    a, probs = device_amps(M, l, 3)
    seed = pb.split_next(1, 0xD1EC7)
    top, direct, st = pb.api.postprocess_device_amps(n, oq, fixed, a.data_ptr(), 512, direct_seed=seed)
    assert np.array_equal(direct, port.direct(n, oq, fixed, probs, seed))
    assert np.array_equal(top, port.top_k(n, oq, fixed, probs, 512))
    # l = 3 (groups smaller than a warp) and l = 7 (two chunks per group)
    for l2, oq2 in ((3, [0, 4, 9]), (7, [0, 1, 2, 3, 4, 5, 6])):
        fixed2, _ = pb.build_candidate_set(n, oq2, 300, 8)
        a2, probs2 = device_amps(300, l2, 11)
        _, d2, _ = pb.api.postprocess_device_amps(n, oq2, fixed2, a2.data_ptr(), 0, direct_seed=seed)
        assert np.array_equal(d2, port.direct(n, oq2, fixed2, probs2, seed))


def test_device_xeb_against_statevector(ref):
    """XEB of both sample sets reduced on the device from a device statevector
    equals the reference xeb with ideal_probability (to the summation order)."""
    import torch
    n, oq, M, l = 16, [0, 1, 2], 256, 3
    g = torch.Generator(device="cuda").manual_seed(0)
    state = torch.randn(1 << n, 2, dtype=torch.float64, device="cuda", generator=g)
    state /= state.norm()
    st_h = state.cpu().numpy()
    q_all = st_h[:, 0] * st_h[:, 0] + st_h[:, 1] * st_h[:, 1]
    fixed, _ = pb.build_candidate_set(n, oq, M, 3)
    amps, probs = device_amps(M, l, 4)
    seed = 77
    top, direct, st = pb.api.postprocess_device_amps(n, oq, fixed, amps.data_ptr(), 64, direct_seed=seed,
                                                     d_state=state.data_ptr())
    for samples, got in ((top, st["xeb_topk"]), (direct, st["xeb_direct"])):
        want = ref.xeb(n, samples, q_all[samples.astype(np.int64)])
        assert abs(got - want) <= 1e-12 * max(1.0, abs(want))
        assert abs(pb.api.xeb_state(n, samples, state.data_ptr()) - want) <= 1e-12 * max(1.0, abs(want))


@pytest.mark.parametrize("order", ["radix", "buckets"])
def test_errors_nan_zero_group_and_signed_zero(ref, order, monkeypatch):
    import torch
    monkeypatch.setenv("RCSG_TOPK_BUCKETS", "0" if order == "radix" else "1")
    n, oq = 8, [0, 1]
    fixed, _ = pb.build_candidate_set(n, oq, 16, 1)
    a = torch.zeros(16 * 4, 2, dtype=torch.float64, device="cuda")
    with pytest.raises(pb.ConfigError, match="zero total probability"):
        pb.api.postprocess_device_amps(n, oq, fixed, a.data_ptr(), 0, direct_seed=1)
    a[5, 0] = float("nan")
    with pytest.raises(pb.ConfigError, match="NaN"):
        pb.api.postprocess_device_amps(n, oq, fixed, a.data_ptr(), 4)
    # -0.0 ranks equal to +0.0; negative ProbFn values rank below zero (reference operator>)
    probs = np.zeros((16, 4))
    probs[::2, 1] = -0.0
    probs[3, 2] = -1e-300
    probs[4, 0] = 1e-3
    for k in (1, 5, 64):
        assert np.array_equal(pb.top_k_select(n, oq, fixed, probs, k), ref.top_k(n, oq, fixed, probs, k))


@pytest.mark.parametrize("slack", [None, "1e9", "1e300"])
def test_direct_running_sum_search_and_exact_chain(slack, monkeypatch):
    """Direct sampling finds the pick by binary search over the left-to-right
    running sums and re-runs the reference's exact subtraction chain when u is
    within the rounding margin of a running sum.  Widening the margin
    (RCSG_DIRECT_SLACK) sends some / every group down the exact chain; the
    samples must equal the reference's either way, on quantised amplitudes
    (exact ties and zero probabilities) and tiny ones (subnormal products)."""
    if slack:
        monkeypatch.setenv("RCSG_DIRECT_SLACK", slack)
    n, oq = 30, [0, 1, 2, 3, 4, 5]
    seed = pb.split_next(3, 0xD1EC7)
    for M, l, quant, scale in ((1 << 15, 6, 2.0**13, 1.0), (4096, 6, None, 2.0**-520), (2000, 5, 2.0**12, 1.0)):
        fixed, _ = pb.build_candidate_set(n, oq[:l], M, 17)
        a, probs = device_amps(M, l, 21, quantize=quant)
        if scale != 1.0:
            a = (a * scale).contiguous()
            h = a.cpu().numpy()
            probs = (h[:, 0] * h[:, 0] + h[:, 1] * h[:, 1]).reshape(M, 1 << l)
        _, d, st = pb.api.postprocess_device_amps(n, oq[:l], fixed, a.data_ptr(), 0, direct_seed=seed)
        assert np.array_equal(d, port.direct(n, oq[:l], fixed, probs, seed)), (M, l, quant, scale)
