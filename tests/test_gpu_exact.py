"""GPU statevector (simulate_exact, statevector.cpp:79-86) against the CPU
oracle's statevector and against the contraction path."""
import numpy as np
import pytest

import paper_2406_18889_b200 as pb
from oracle import port

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("spec", [(12, 8, "grid(3,4)", 1), (10, 12, "line", 7), (16, 10, "grid(4,4)", 3)])
def test_statevector_matches_oracle_bit_for_bit(spec):
    import torch
    n, cycles, topo, seed = spec
    p = pb.Problem(n, cycles, topo, seed, [0, 1, 2], 1 << 30, "low").build()
    want = port.statevector(n, p.gates())
    state = torch.empty(1 << n, dtype=torch.complex128, device="cuda")
    p.exact_state_device(state.data_ptr())
    got = state.cpu().numpy()
    # separately rounded products and sums in the reference's order
    assert np.array_equal(got, want), np.max(np.abs(got - want))


def test_exact_probabilities_match_contraction():
    p = pb.Problem(12, 8, "grid(3,4)", 1, [0, 1, 2], 1 << 30, "low").build()
    fixed, _ = pb.build_candidate_set(12, [0, 1, 2], 16, pb.split_next(1, 0xCA11D))
    amps = p.contract_groups(fixed, precision="f64", configs=None)
    idx = [pb.member(12, [0, 1, 2], int(f), i) for f in fixed for i in range(8)]
    probs = p.exact_probabilities(idx)
    assert np.allclose(probs, (np.abs(amps) ** 2).reshape(-1), rtol=1e-10, atol=1e-16)


def test_statevector_30_qubits_norm():
    """cfg2's circuit (n = 30, 17 GB of complex f64): the state stays normalised."""
    import torch
    p = pb.Problem(30, 14, "grid(5,6)", 1, list(range(6)), 3 << 30, "low").build()
    state = torch.empty(1 << 30, dtype=torch.complex128, device="cuda")
    p.exact_state_device(state.data_ptr())
    norm = float(torch.sum(state.real ** 2 + state.imag ** 2))
    assert abs(norm - 1.0) < 1e-9


def test_statevector_rejects_bad_input():
    """Capacity and configuration errors, like simulate_exact / apply_gate
    (statevector.cpp:79-82): CapacityError above the cap, ConfigError for bad
    gate targets."""
    import ctypes as C
    import torch
    from paper_2406_18889_b200 import _native
    lib = _native.lib()
    state = torch.empty(16, dtype=torch.complex128, device="cuda")
    nt = (C.c_int32 * 1)(2)
    tg = (C.c_int32 * 2)(1, 1)  # a two-qubit gate on the same qubit twice
    u = (C.c_double * 32)(*([1.0] + [0.0] * 31))
    assert lib.rcsg_statevector(4, 1, nt, tg, u, C.c_void_p(state.data_ptr())) == _native.RCSG_ERR_CONFIG
    tg2 = (C.c_int32 * 2)(0, 7)  # target outside the register
    assert lib.rcsg_statevector(4, 1, nt, tg2, u, C.c_void_p(state.data_ptr())) == _native.RCSG_ERR_CONFIG
    assert lib.rcsg_statevector(40, 0, nt, tg, u, C.c_void_p(state.data_ptr())) == _native.RCSG_ERR_CAPACITY
