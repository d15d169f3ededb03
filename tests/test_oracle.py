"""Pins the CPU checker (oracle/port, plain-C restatement) against the
reference's own outputs: the committed golden fixtures (tests/golden/, made by
make_golden.py from the unmodified reference library) and, when it is built,
the reference library itself.  Bit-exact: same algorithm, same summation order."""
import os

import numpy as np
import pytest

from oracle import port

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
CASES = ["cfg1", "sliced_line10", "broken_ring10", "grid44_sliced_broken"]


def load(name):
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))


def net_plan(g):
    net = dict(leaf_rank=g["leaf_rank"], leaf_labels=g["leaf_labels"], leaf_data=g["leaf_data"],
               n_labels=int(g["n_labels"]), n_qubits=len(g["output_labels"]), output_labels=g["output_labels"],
               open_labels=g["open_labels"], open_qubits=g["open_qubits"])
    plan = dict(steps=g["steps"], sliced=g["sliced"], broken=g["broken"])
    return net, plan


@pytest.fixture(scope="module", autouse=True)
def need_port():
    if not port.available():
        pytest.skip("oracle/_ref/librcs_port.so not built")


@pytest.mark.parametrize("name", CASES)
def test_port_amplitudes_bit_exact_vs_reference_fixture(name):
    g = load(name)
    pn = port.PortNet(*net_plan(g))
    configs = g["configs"] if len(g["broken"]) else None
    for i, fb in enumerate(g["group_fixed"]):
        got = pn.contract_group(int(fb), configs=configs)
        assert np.array_equal(got.view(np.float64), g["amplitudes"][i].view(np.float64)), (name, i)


@pytest.mark.parametrize("name", CASES)
def test_port_statevector_vs_reference_fixture(name):
    g = load(name)
    if "statevector" not in g:
        pytest.skip("no statevector")
    n = len(g["output_labels"])
    sv = port.statevector(n, g["gates"])
    assert np.array_equal(sv, g["statevector"])


def test_port_sampler_vs_reference_fixture():
    s = load("sampler")
    for k in (1, 7, 64, 512, 4096):
        assert np.array_equal(port.top_k(12, [0, 1, 2], s["fixed"], s["probs"], k), s[f"topk_{k}"])
    for k in (1, 100, 512):
        assert np.array_equal(port.top_k(9, [1, 4, 7], s["fixed_ties"], s["ties"], k), s[f"ties_{k}"])
    assert np.array_equal(port.direct(12, [0, 1, 2], s["fixed"], s["probs"], int(s["direct_seed"])), s["direct"])
    assert port.xeb(12, s["q"]) == s["xeb"]
    for idx, key in s["lexkeys"]:
        assert port.lexkey(int(idx), 12) == int(key)
    assert port.split_next(1, 0xCA11D) == int(s["split_ca11d"])
    fixed, dup = port.candidates(12, [0, 1, 2], 512, int(s["split_ca11d"]))
    assert np.array_equal(fixed, s["fixed"]) and dup == int(s["duplicate_groups"])


def test_port_known_answers():
    # test_sampling.cpp:111-128 (ties -> {0, 2}), :242-265 (lexicographic keys)
    assert list(port.top_k(2, [0, 1], [0], np.full((1, 4), 0.25), 2)) == [0, 2]
    assert port.lexkey(1, 4) == 8 and port.lexkey(8, 4) == 1 and port.lexkey(0b0110, 4) == 0b0110
    # Gray-code configurations: distinct, one-bit steps (test_contraction.cpp:95-116)
    cf = port.broken_configs(6, 64, 5)
    assert len(set(cf.tolist())) == 64
    part = port.broken_configs(6, 6, 5)
    for a, b in zip(part[:-1], part[1:]):
        d = int(a) ^ int(b)
        assert d and d & (d - 1) == 0
    with pytest.raises(port.PortError):
        port.broken_configs(6, 65, 1)


def test_port_numeric_fault_step():
    inf = float("inf")
    net = dict(leaf_rank=[2, 1], leaf_labels=[0, 1, 1], leaf_data=np.array([inf, 0, 0, 0, 0, 0, 1, 0, 1, 0, 1, 0.0]),
               n_labels=2, n_qubits=1, output_labels=[0], open_labels=[0], open_qubits=[0])
    pn = port.PortNet(net, dict(steps=np.array([[0, 1, 2, 0, 0, 0]]), sliced=[], broken=[]))
    with pytest.raises(port.PortError) as e:
        pn.execute({})
    assert e.value.code == 3 and e.value.step == 0


def test_port_vs_live_reference(ref):
    """When the reference library is built, the restatement agrees bit for bit."""
    p = ref.RefProblem(12, 8, "grid(3,4)", 1, [0, 1, 2], 1 << 30, "low").build()
    pn = port.PortNet(p.net, p.plan)
    fixed, _ = ref.candidates(12, [0, 1, 2], 8, ref.split_next(1, 0xCA11D))
    for fb in fixed:
        assert np.array_equal(pn.contract_group(int(fb)), p.contract_group(int(fb)))
    q = ref.RefProblem(10, 10, "line", 17, [0, 3, 5, 8], 20000, "low").build()
    qn = port.PortNet(q.net, q.plan)
    for s in (0, 5):
        a = {**{int(k): v for k, v in zip(q.plan["sliced"], [(s >> b) & 1 for b in range(len(q.plan["sliced"]))])}}
        fixed_q = [x for x in range(10) if x not in (0, 3, 5, 8)]
        for b, qq in enumerate(fixed_q):
            a[int(q.net["output_labels"][qq])] = (0b101001 >> b) & 1
        assert np.array_equal(qn.execute(a), q.execute(a))
