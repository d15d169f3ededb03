"""Artifact formats against the reference's own writers:
plan.json equal as JSON to plan_to_json (contraction_plan.cpp:451-491) and
importable in both directions, timings.csv (contraction_engine.cpp:347-354)
and samples.txt (sampling.cpp:177-210) byte-identical.  CPU only.

plan.json is compared as parsed JSON: the oracle build links the nlohmann/json
copy vendored in the cudnn_frontend wheel, which prints integer arrays on one
line; upstream nlohmann (and our writer) pretty-prints every array."""
import json

import numpy as np
import pytest

import paper_2406_18889_b200 as pb


def test_plan_json_matches_reference(ref):
    for spec in [(12, 8, "grid(3,4)", 1, [0, 1, 2], 1 << 30, "low"),
                 (30, 14, "grid(5,6)", 1, list(range(6)), 3 << 30, "low"),
                 (10, 10, "ring", 62, list(range(10)), 1 << 30, "low", 5, 16)]:
        mine = pb.Problem(*spec).build().plan_json()
        theirs = ref.RefProblem(*spec).build().plan_json()
        assert json.loads(mine) == json.loads(theirs), spec
        assert mine.startswith('{\n  "broken": [')  # dump(2) layout, keys sorted


def test_plan_import_round_trip_and_scale_plans():
    spec = (30, 14, "grid(5,6)", 1, list(range(6)), 3 << 30, "low")
    p = pb.Problem(*spec).build()
    q = pb.Problem(*spec).build(planner="scale", trials=16)
    text = q.plan_json()
    d = json.loads(text)
    assert d["totals"]["n_slices"] == q.n_slices
    p.import_plan(text)  # the scale plan, imported into another handle
    assert np.array_equal(p.plan["steps"], q.plan["steps"])
    assert list(p.plan["sliced"]) == list(q.plan["sliced"])
    assert p.plan["flops_per_slice"] == q.plan["flops_per_slice"]
    assert p.plan_json() == text


def test_plan_import_from_reference_json(ref):
    spec = (12, 8, "grid(3,4)", 1, [0, 1, 2], 1 << 12, "low")
    r = ref.RefProblem(*spec).build()
    p = pb.Problem(12, 8, "grid(3,4)", 1, [0, 1, 2], 1 << 30, "low").build()
    p.import_plan(r.plan_json())
    assert np.array_equal(p.plan["steps"][:, :3], r.plan["steps"][:, :3])
    assert list(p.plan["sliced"]) == list(r.plan["sliced"])
    assert p.plan["flops_per_slice"] == r.plan["flops_per_slice"]
    assert p.plan["peak_bytes"] == r.plan["peak_bytes"]


def test_timings_csv_and_samples_text_match_reference(ref):
    ids, bits = [0, 1, 2], [5, 4, 6]
    ms, flops = [1.25, 0.000123456789, 12345.678], [10, 2 ** 40, 7]
    assert pb.api.timings_to_csv(ids, bits, ms, flops) == ref.timings_csv(ids, bits, ms, flops)
    s = np.array([19, 0, 31, 5], np.uint64)
    for topk, k in ((False, 0), (True, 4)):
        text = pb.api.samples_to_text(5, s, topk, k)
        assert text == ref.samples_text(5, topk, k, s)
        n, tk, kk, back = pb.api.samples_from_text(text)
        assert (n, tk, kk) == (5, topk, k) and np.array_equal(back, s)
    assert pb.api.samples_to_text(5, [19]).splitlines()[-1] == "11001"  # test_sampling.cpp:242-258


def test_state_fidelity_and_predicted_topk_xeb():
    """state_fidelity (contraction_engine.cpp:327-345) and predicted_topk_xeb
    (sampling.cpp:147-151), host-side, against their closed forms."""
    rng = np.random.default_rng(3)
    e = rng.normal(size=64) + 1j * rng.normal(size=64)
    a = 0.7 * e + 0.3 * (rng.normal(size=64) + 1j * rng.normal(size=64))
    want = abs(np.vdot(e, a)) ** 2 / (np.vdot(a, a).real * np.vdot(e, e).real)
    got, warn = pb.api.state_fidelity(a, e)
    assert abs(got - want) < 1e-14 and not warn
    assert pb.api.state_fidelity(e * 2j, e)[0] == pytest.approx(1.0, abs=1e-14)
    assert pb.api.state_fidelity(np.zeros(64), e) == (0.0, True)  # zero-norm approximation -> 0 + warning
    with pytest.raises(pb.ConfigError):
        pb.api.state_fidelity(np.ones(4), np.zeros(4))  # exact collection of zero norm
    with pytest.raises(pb.ConfigError):
        pb.api.state_fidelity(np.ones(4), np.ones(8))
    assert abs(pb.api.predicted_topk_xeb(1.0, 1 << 30, 1 << 15) - 10.3972) <= 1e-4  # acceptance.cpp:224-226
    with pytest.raises(pb.ConfigError):
        pb.api.predicted_topk_xeb(1.0 + 1e-12, 100, 10)  # F > 1 rejected


@pytest.mark.parametrize("name", ["cfg3", "cfg4", "cfg5"])
def test_committed_bench_plans_import(name):
    """The bench's cfg3-5 plans (plans/<cfg>.json, found offline by the scale
    planner, tools/plan_search.py) import onto the circuit they were planned for
    and export byte-identically; the slice count matches the planner report."""
    import json
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    meta = json.load(open(os.path.join(root, "plans", f"{name}.meta.json")))
    n, m, topo = {"cfg3": (53, 12, "sycamore53"), "cfg4": (53, 20, "sycamore53"),
                  "cfg5": (60, 24, "zuchongzhi60")}[name]
    text = open(os.path.join(root, "plans", f"{name}.json")).read()
    p = pb.Problem(n, m, topo, 1, list(range(6)), meta["budget_bytes"], "low").build(plan_json=text)
    assert len(p.plan["sliced"]) == meta["report"]["n_sliced"]
    assert p.plan_json() == text
