"""Host-side inputs of the hot path (C++ in the product library): circuits,
networks, plans and candidate sets must be bit-identical to the reference's,
so the GPU runs exactly the reference's plan.  Checked against the golden
fixtures (always) and the live reference library (when built).  CPU only."""
import os

import numpy as np
import pytest

import paper_2406_18889_b200 as pb

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
CASES = ["cfg1", "sliced_line10", "broken_ring10", "grid44_sliced_broken"]


def load(name):
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))


@pytest.mark.parametrize("name", CASES)
def test_pipeline_bit_identical_to_reference_fixture(name):
    g = load(name)
    spec = eval(str(g["spec"]))  # the fixture's own (n, cycles, topology, seed, open, budget, effort, K, m)
    p = pb.Problem(*spec).build()
    assert np.array_equal(p.gates(), g["gates"])
    assert np.array_equal(p.net["leaf_rank"], g["leaf_rank"])
    assert np.array_equal(p.net["leaf_labels"], g["leaf_labels"])
    assert np.array_equal(p.net["leaf_data"], g["leaf_data"])
    assert p.net["label_names"] == list(g["label_names"])
    for k in ("steps", "sliced", "broken", "fixed_outputs", "configs"):
        assert np.array_equal(p.plan[k], g[k]), k
    tot = g["totals"]
    assert (p.plan["flops_per_slice"], p.plan["traffic_bytes_per_slice"], p.plan["peak_bytes"],
            p.plan["memory_budget_bytes"]) == tuple(int(x) for x in tot)
    if len(spec[4]) < spec[0]:
        fixed, dup = pb.build_candidate_set(spec[0], spec[4], len(g["group_fixed"]), pb.split_next(spec[3], 0xCA11D))
        assert np.array_equal(fixed, g["group_fixed"]) and dup == int(g["duplicate_groups"])


def test_cfg2_plan_has_256_slices():
    # BASELINE configs[1]: 30 qubits, 14 cycles, l = 6, 2^8 slices at budget 3*2^30 B
    p = pb.Problem(30, 14, "grid(5,6)", 1, list(range(6)), 3 << 30, "low").build()
    assert len(p.plan["sliced"]) == 8
    assert p.plan["flops_per_slice"] == 367686457536
    assert len(p.plan["steps"]) == 621


@pytest.mark.parametrize("spec", [
    (8, 8, "line", 73, [1, 3], 1 << 30, "medium", 0, 1),
    (14, 10, "line", 3, [0, 1, 2, 3], 1 << 14, "low", 0, 1),  # deep slicing, rank-0 tensors
    (12, 12, "ring", 5, list(range(12)), 1 << 30, "low", 4, 3),
    (16, 10, "grid(4,4)", 3, [0, 1, 2, 3], 1 << 16, "medium", 3, 5),
])
def test_planner_matches_live_reference(ref, spec):
    r = ref.RefProblem(*spec).build()
    m = pb.Problem(*spec).build()
    for k in ("steps", "sliced", "broken", "fixed_outputs", "configs"):
        assert np.array_equal(r.plan[k], m.plan[k]), k
    assert r.plan["peak_bytes"] == m.plan["peak_bytes"]
    assert r.net["label_names"] == m.net["label_names"]


def test_sampler_host_pieces_vs_fixture():
    s = load("sampler")
    assert pb.split_next(1, 0xCA11D) == int(s["split_ca11d"])
    assert pb.split_next(1, 0xD1EC7) == int(s["split_d1ec7"])
    fixed, dup = pb.build_candidate_set(12, [0, 1, 2], 512, int(s["split_ca11d"]))
    assert np.array_equal(fixed, s["fixed"]) and dup == int(s["duplicate_groups"])
    for idx, key in s["lexkeys"]:
        assert pb.lexkey(int(idx), 12) == int(key)
    # xeb is reduced on the device (tests/test_gpu_sampling.py checks it against this fixture's value)


def test_candidate_set_structure_and_validation():
    # test_sampling.cpp:30-66
    fixed, _ = pb.build_candidate_set(4, [0, 1], 3, 77)
    for fb in fixed:
        members = [pb.member(4, [0, 1], int(fb), i) for i in range(4)]
        assert len({m & 0b0011 for m in members}) == 4 and len({m & 0b1100 for m in members}) == 1
    a, _ = pb.build_candidate_set(12, list(range(12)), 1, 1)
    b, _ = pb.build_candidate_set(12, list(range(12)), 1, 999)
    assert np.array_equal(a, b)
    for bad in (([0, 0], 1), ([5], 1), ([0, 1, 2, 3], 2), ([0], 0)):
        with pytest.raises(pb.ConfigError):
            pb.build_candidate_set(4, bad[0], bad[1], 0)
    _, dup = pb.build_candidate_set(3, [0, 1], 8, 5)
    assert dup >= 6


def test_broken_configs_and_errors():
    cf = pb.broken_configs(6, 64, 5)
    assert sorted(cf.tolist()) == list(range(64))
    with pytest.raises(pb.ConfigError):
        pb.broken_configs(6, 0, 1)
    with pytest.raises(pb.ConfigError):
        pb.broken_configs(6, 65, 1)


def test_infeasible_budget_and_bad_open_qubits():
    with pytest.raises(pb.ConfigError):
        pb.Problem(8, 8, "line", 3, list(range(8)), 100, "low").build()
    with pytest.raises(pb.ConfigError):
        pb.Problem(4, 2, "line", 1, [0, 0], 1 << 30, "low").build()
    with pytest.raises(pb.ConfigError):
        pb.Problem(4, 2, "line", 1, [4], 1 << 30, "low").build()


def test_sycamore53_topology():
    p = pb.Problem(53, 2, "sycamore53", 1, list(range(6)), 1 << 40, "low").build()
    g = p.gates()
    two = g[g[:, 3] >= 0]
    assert len(two) > 0 and two[:, 2:].max() < 53
    for layer in np.unique(two[:, 0]):
        qs = two[two[:, 0] == layer][:, 2:].reshape(-1)
        assert len(set(qs.tolist())) == len(qs)  # disjoint couplers per layer
