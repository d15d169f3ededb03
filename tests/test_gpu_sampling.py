"""GPU post-processing parity: top-k order, direct-sample indices and XEB must be
bit-identical to the reference sampler (oracle/_ref) on identical probabilities."""
import numpy as np
import pytest

import paper_2406_18889_b200 as pb
from oracle import port

pytestmark = pytest.mark.gpu


def probs_for(fixed, l, seed, n=12, open_q=(0, 1, 2)):
    # a function of the bitstring index, like the reference's ProbFn
    rng = np.random.default_rng(seed)
    table = rng.exponential(size=1 << n) / 2**n
    return np.array([[table[pb.member(n, list(open_q), int(f), i)] for i in range(1 << l)] for f in fixed])


@pytest.mark.parametrize("k", [1, 7, 64, 512, 4096])
def test_topk_bit_exact(ref, k):
    fixed, _ = ref.candidates(12, [0, 1, 2], 512, ref.split_next(1, 0xCA11D))
    probs = probs_for(fixed, 3, k)
    got = pb.top_k_select(12, [0, 1, 2], fixed, probs, k)
    want = ref.top_k(12, [0, 1, 2], fixed, probs, k)
    assert np.array_equal(got, want)


def test_topk_ties_lexicographic(ref):
    # test_sampling.cpp:111-128: flat 2-qubit -> {0, 2}
    got = pb.top_k_select(2, [0, 1], [0], np.full((1, 4), 0.25), 2)
    assert list(got) == [0, 2]
    probs = np.full((64, 8), 1.0 / 512)  # many ties and duplicate groups
    fixed, _ = ref.candidates(9, [1, 4, 7], 64, 5)
    for k in (1, 100, 512):
        assert np.array_equal(pb.top_k_select(9, [1, 4, 7], fixed, probs, k),
                              ref.top_k(9, [1, 4, 7], fixed, probs, k))


def test_topk_range_errors():
    with pytest.raises(pb.ConfigError):
        pb.top_k_select(2, [0, 1], [0], np.full((1, 4), 0.25), 0)
    with pytest.raises(pb.ConfigError):
        pb.top_k_select(2, [0, 1], [0], np.full((1, 4), 0.25), 5)


def test_direct_sample_bit_exact(ref):
    fixed, _ = ref.candidates(20, [0, 5, 9, 13], 4096, 77)
    probs = probs_for(fixed, 4, 3, n=20, open_q=(0, 5, 9, 13))
    seed = ref.split_next(1, 0xD1EC7)
    assert np.array_equal(pb.direct_sample(20, [0, 5, 9, 13], fixed, probs, seed),
                          ref.direct(20, [0, 5, 9, 13], fixed, probs, seed))


def test_direct_sample_spike_and_zero_group():
    fixed, _ = pb.build_candidate_set(6, [0, 1], 64, 9)
    spiked = np.zeros((64, 4))
    spiked[:, 0] = 1.0
    s = pb.direct_sample(6, [0, 1], fixed, spiked, 4)
    assert all(int(x) == pb.member(6, [0, 1], int(f), 0) for x, f in zip(s, fixed))
    with pytest.raises(pb.ConfigError, match="group 0"):
        pb.direct_sample(6, [0, 1], fixed, np.zeros((64, 4)), 4)


def test_xeb_matches_reference(ref):
    q = np.random.default_rng(0).exponential(size=1000) / 4096
    samples = np.arange(1000, dtype=np.uint64)
    # the reference sums sequentially; the device reduction is fixed-order (tree)
    assert ref.xeb(12, samples, q) == port.xeb(12, q)
    assert abs(pb.xeb(12, q) - ref.xeb(12, samples, q)) <= 1e-13 * abs(ref.xeb(12, samples, q))
    assert pb.xeb(12, [1 / 4096]) == 0.0
    import os
    g = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", "sampler.npz")))
    assert abs(pb.xeb(12, g["q"]) - float(g["xeb"])) <= 1e-13 * abs(float(g["xeb"]))
    with pytest.raises(pb.ConfigError):
        pb.xeb(12, [-0.5])


def test_topk_from_device_amplitudes_matches_port():
    import torch
    p = pb.Problem(12, 8, "grid(3,4)", 1, [0, 1, 2], 1 << 30, "low").build()
    fixed, _ = pb.build_candidate_set(12, [0, 1, 2], 512, pb.split_next(1, 0xCA11D))
    acc = torch.zeros(512 * 8 * 2, dtype=torch.float64, device="cuda")
    p.contract_groups_device(fixed, acc.data_ptr(), precision="f64", configs=None)
    amps = acc.cpu().numpy().view(np.complex128).reshape(512, 8)
    probs = amps.real * amps.real + amps.imag * amps.imag
    for k in (1, 64, 4096):
        got = pb.api.top_k_from_device_amps(12, [0, 1, 2], fixed, acc.data_ptr(), k)
        assert np.array_equal(got, port.top_k(12, [0, 1, 2], fixed, probs, k))
    seed = pb.split_next(1, 0xD1EC7)
    got = pb.api.direct_from_device_amps(12, [0, 1, 2], fixed, acc.data_ptr(), seed)
    assert np.array_equal(got, port.direct(12, [0, 1, 2], fixed, probs, seed))


@pytest.mark.parametrize("precision", ["tf32", "bf16", "f16"])
def test_topk_reduced_precision_matches_oracle_away_from_ties(precision):
    """Top-k over reduced-precision GPU amplitudes against the f64 oracle's top-k
    (selected bitstrings bit-exact wherever probabilities are not tied
    within the precision's tolerance).  eps = the largest probability error of the
    run; two picks are tied when their oracle probabilities differ by <= 2 eps."""
    import torch
    n, oq, M = 12, [0, 1, 2], 512
    p = pb.Problem(n, 8, "grid(3,4)", 1, oq, 1 << 30, "low").build()
    fixed, _ = pb.build_candidate_set(n, oq, M, pb.split_next(1, 0xCA11D))
    pn = port.PortNet(p.net, p.plan)
    want = np.array([pn.contract_group(int(f)) for f in fixed])
    p_ref = np.abs(want) ** 2
    acc = torch.zeros(M * 8 * 2, dtype=torch.float64, device="cuda")
    p.contract_groups_device(fixed, acc.data_ptr(), precision=precision, configs=None)
    got = acc.cpu().numpy().view(np.complex128).reshape(M, 8)
    eps = np.abs(np.abs(got) ** 2 - p_ref).max()
    assert eps < {"tf32": 1e-2, "f16": 1e-2, "bf16": 1e-1}[precision] * p_ref.max()
    prob_of = {pb.member(n, oq, int(f), i): p_ref[g, i] for g, f in enumerate(fixed) for i in range(8)}
    allp = np.array(sorted(prob_of.values()))
    exact = 0
    for k in (1, 16, 64, 256):
        sel = pb.api.top_k_from_device_amps(n, oq, fixed, acc.data_ptr(), k)
        ref_sel = port.top_k(n, oq, fixed, p_ref, k)
        for a, b in zip(sel, ref_sel):
            pa, pb_ = prob_of[int(a)], prob_of[int(b)]
            assert abs(pa - pb_) <= 2 * eps, (k, a, b)
            # isolated oracle probability (no other bitstring within 2 eps): the pick is exact
            lo, hi = np.searchsorted(allp, pb_ - 2 * eps), np.searchsorted(allp, pb_ + 2 * eps, side="right")
            if hi - lo == 1:
                assert a == b, (k, a, b)
                exact += 1
    assert exact > 0
