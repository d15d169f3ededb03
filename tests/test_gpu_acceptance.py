"""The reference's XEB acceptance criteria (tests/acceptance.cpp:159-231), run
through the GPU pipeline: group-batched contraction with broken edges, the
fused post-processing kernel, and XEB reduced on the device against the exact
GPU statevector (bit-identical to the reference's simulate_exact).

criterion 3 (:159-197): n = 14 line circuits, 10 seeds, K = 1..4 broken edges
  (m = 1), M = 2^16 candidate groups with l = 4: mean direct-sample XEB over
  mean fidelity in [0.7, 1.3] for every K;
criterion 4 (:199-231): n = 16 line circuits, 3 seeds, exhaustive candidates:
  mean top-k XEB / (-ln alpha) in [0.9, 1.1] for k = 2^8..2^14, and
  predicted_topk_xeb(1, 2^30, 2^15) = 10.3972."""
import numpy as np
import pytest

import paper_2406_18889_b200 as pb

pytestmark = pytest.mark.gpu


def test_criterion3_direct_sampling_xeb_tracks_fidelity():
    import torch
    n, open_q, M = 14, [0, 1, 2, 3], 1 << 16
    xeb_k = {K: [] for K in range(1, 5)}
    fid_k = {K: [] for K in range(1, 5)}
    for s in range(1, 11):
        seed = 600 + s
        state = torch.empty(1 << n, dtype=torch.complex128, device="cuda")
        for K in range(1, 5):
            p = pb.Problem(n, n, "line", seed, open_q, 1 << 40, "low", K, 1).build()
            if K == 1:
                p.exact_state_device(state.data_ptr())
                exact = state.cpu().numpy()
            # full approximate state: all 2^(n-l) prefixes
            allp = np.arange(1 << (n - len(open_q)), dtype=np.uint64)
            amps = p.contract_groups(allp, precision="f64")
            full = np.zeros(1 << n, np.complex128)
            idx = np.array([[pb.member(n, open_q, int(f), i) for i in range(16)] for f in allp], np.int64)
            full[idx.reshape(-1)] = amps.reshape(-1)
            fid_k[K].append(pb.api.state_fidelity(full, exact)[0])
            fixed, _ = pb.build_candidate_set(n, open_q, M, pb.split_next(seed, 0xCA11D))
            acc = torch.zeros(M * 16 * 2, dtype=torch.float64, device="cuda")
            p.contract_groups_device(fixed, acc.data_ptr(), precision="f64")
            _, _, st = pb.api.postprocess_device_amps(n, open_q, fixed, acc.data_ptr(), 0,
                                                      direct_seed=pb.split_next(seed, 0xD1EC7) + K,
                                                      d_state=state.data_ptr())
            xeb_k[K].append(st["xeb_direct"])
    ratios = [np.mean(xeb_k[K]) / np.mean(fid_k[K]) for K in range(1, 5)]
    print("XEB / F per K:", ratios)
    assert all(0.7 <= r <= 1.3 for r in ratios), ratios


def test_criterion4_ideal_topk_amplification_law():
    import torch
    n = 16
    ratio = {lk: 0.0 for lk in range(8, 15)}
    for s in range(3):
        p = pb.Problem(n, n, "line", 4242 + s, list(range(n)), 1 << 40, "low").build()
        state = torch.empty(1 << n, dtype=torch.complex128, device="cuda")
        p.exact_state_device(state.data_ptr())
        for lk in range(8, 15):
            k = 1 << lk
            # exhaustive candidate set (l = n, one group): the amplitudes ARE the statevector
            top, _, st = pb.api.postprocess_device_amps(n, list(range(n)), [0], state.data_ptr(), k,
                                                        d_state=state.data_ptr())
            ratio[lk] += st["xeb_topk"] / -np.log(k / 65536.0) / 3
    print("XEB_topk / -ln(alpha):", ratio)
    assert all(0.9 <= r <= 1.1 for r in ratio.values()), ratio
    assert abs(pb.api.predicted_topk_xeb(1.0, 1 << 30, 1 << 15) - 10.3972) <= 1e-4
