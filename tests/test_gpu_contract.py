"""GPU parity of the contraction path against the CPU oracle (reference library
oracle/_ref and the C restatement oracle/port), on the same circuits, seeds and
plans.  Tolerances are norm-wise relative error per group, per precision mode
(SURVEY §8c): f64 1e-10, f32 1e-5, tf32 1e-2, 3xtf32 1e-5.
"""
import numpy as np
import pytest

import paper_2406_18889_b200 as pb
from oracle import port

pytestmark = pytest.mark.gpu

TOL = {"f64": 1e-10, "f32": 2e-5, "tf32": 1e-2, "3xtf32": 2e-5, "bf16": 1.5e-1, "f16": 1e-2}


def rel(a, b):
    a = np.asarray(a).reshape(-1)
    b = np.asarray(b).reshape(-1)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def cfg1(M=64):
    p = pb.Problem(12, 8, "grid(3,4)", 1, [0, 1, 2], 1 << 30, "low").build()
    fixed, _ = pb.build_candidate_set(12, [0, 1, 2], M, pb.split_next(1, 0xCA11D))
    return p, fixed


@pytest.mark.parametrize("precision", ["f64", "f32", "tf32", "3xtf32", "bf16", "f16"])
def test_cfg1_groups_match_oracle(precision):
    p, fixed = cfg1(64)
    pn = port.PortNet(p.net, p.plan)
    got = p.contract_groups(fixed, precision=precision)
    for g, fb in enumerate(fixed):
        want = pn.contract_group(int(fb))
        assert rel(got[g], want) < TOL[precision], (g, rel(got[g], want))


def test_cfg1_group_batching_equals_single_groups():
    p, fixed = cfg1(128)
    batch = p.contract_groups(fixed)
    for g in range(0, 128, 17):
        single = p.contract_group(int(fixed[g]))
        assert rel(batch[g], single) < 1e-13


def test_sliced_plan_matches_oracle_and_slice_sum():
    p = pb.Problem(10, 10, "line", 17, [0, 3, 5, 8], 20000, "low").build()
    assert len(p.plan["sliced"]) >= 3
    pn = port.PortNet(p.net, p.plan)
    fixed = np.array([0, 5, 22, 63], np.uint64)
    got = p.contract_groups(fixed)
    for g, fb in enumerate(fixed):
        assert rel(got[g], pn.contract_group(int(fb))) < 1e-10
    # linearity over disjoint slice ranges
    half = p.n_slices // 2
    a = p.contract_groups(fixed, slices=(0, half))
    b = p.contract_groups(fixed, slices=(half, p.n_slices))
    assert rel(a + b, got) < 1e-12


def test_broken_edges_path_sum_matches_oracle():
    p = pb.Problem(10, 10, "ring", 62, list(range(10)), 1 << 30, "low", 5, 16).build()
    pn = port.PortNet(p.net, p.plan)
    want = pn.contract_group(0, configs=p.plan["configs"])
    got = p.contract_groups([0])[0]
    assert rel(got, want) < 1e-10
    amps, flops = p.contract(configs="all")
    assert rel(amps, want) < 1e-10
    assert flops == p.plan["flops_per_slice"] * p.n_slices * len(p.plan["configs"])


def test_complete_path_sum_reproduces_exact():
    # test_contraction.cpp:55-67 — summing all 2^K configurations is exact
    for K in (2, 4):
        p = pb.Problem(10, 10, "line", 40 + K, list(range(10)), 1 << 30, "low", K, 1 << K).build()
        exact = pb.Problem(10, 10, "line", 40 + K, list(range(10)), 1 << 30, "low").build()
        full = exact.contract_groups([0], configs=None)[0]
        summed = p.contract_groups([0])[0]
        assert rel(summed, full) < 1e-10


def test_contract_group_matches_statevector_slice():
    # test_tensor_network.cpp:84-109 / test_contraction.cpp:174-198
    n = 12
    p = pb.Problem(n, n, "line", 31, [0, 2, 5, 7], 1 << 30, "low").build()
    sv = port.statevector(n, p.gates())
    fixed_q = [q for q in range(n) if q not in (0, 2, 5, 7)]
    for fb in (0, 0b101101, (1 << len(fixed_q)) - 1):
        amps = p.contract_group(fb)
        for i in range(16):
            full = sum(1 << q for j, q in enumerate((0, 2, 5, 7)) if (i >> j) & 1)
            full |= sum(1 << q for b, q in enumerate(fixed_q) if (fb >> b) & 1)
            assert abs(amps[i] - sv[full]) <= 1e-8 * max(abs(sv[full]), 1e-14)


def test_execute_assignment_matches_oracle():
    p = pb.Problem(10, 10, "line", 17, [0, 3, 5, 8], 20000, "low").build()
    pn = port.PortNet(p.net, p.plan)
    for s in (0, 3, p.n_slices - 1):
        a = p.assignment_gsc(0b101001, s)
        assert rel(p.execute(a), pn.execute(a)) < 1e-10


def test_numeric_fault_reports_step():
    inf = float("inf")
    net = dict(leaf_rank=[2, 1], leaf_labels=[0, 1, 1], leaf_data=[inf, 0, 0, 1, 1, 1], n_labels=2,
               n_qubits=1, output_labels=[0], open_labels=[0], open_qubits=[0])
    with pytest.raises(pb.NumericFault) as e:
        pb.execute_desc(net, [(0, 1, 2)], [-1, -1])
    assert e.value.step_index == 0 and e.value.exit_code == 3


def test_two_by_two_product_layout():
    # test_tensor_network.cpp:147-178: output index (c<<1)|a
    A = [1, 2j, -1 + 1j, 3]
    B = [1j, 2, 1 - 1j, 0]
    net = dict(leaf_rank=[2, 2], leaf_labels=[0, 1, 1, 2], leaf_data=A + B, n_labels=3, n_qubits=2,
               output_labels=[0, 2], open_labels=[0, 2], open_qubits=[0, 1])
    out = pb.execute_desc(net, [(0, 1, 2)], [-1, -1, -1])
    for a in range(2):
        for c in range(2):
            want = A[a * 2] * B[c] + A[a * 2 + 1] * B[2 + c]
            assert abs(out[(c << 1) | a] - want) < 1e-12


def test_empty_circuit_scalar():
    # test_tensor_network.cpp:43-61 — three |0> caps, all outputs pinned
    p = pb.Problem.from_network([1, 1, 1], [0, 1, 2], [1, 0, 1, 0, 1, 0], ["q0.in", "q1.in", "q2.in"],
                                3, [0, 1, 2], [], [])
    assert p.contract_groups([0], configs=None)[0][0] == pytest.approx(1.0)
    assert abs(p.contract_groups([0b010], configs=None)[0][0]) < 1e-12


def test_error_taxonomy():
    p = pb.Problem(6, 6, "line", 9, list(range(6)), 1 << 30, "low").build()
    with pytest.raises(pb.ConfigError):
        p.execute({9999: 0})
    with pytest.raises(pb.ConfigError):
        p.execute({0: 2})
    with pytest.raises(pb.ConfigError):  # exact contraction of a plan with broken edges
        q = pb.Problem(6, 6, "line", 9, list(range(6)), 1 << 30, "low", 2, 2).build()
        q.contract_groups([0], configs=None)


# ---- against the reference's own outputs (golden fixtures, tests/golden/) -----
GOLDEN_CASES = ["cfg1", "sliced_line10", "broken_ring10", "grid44_sliced_broken"]


@pytest.mark.parametrize("precision", ["f64", "tf32", "bf16", "f16"])
@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_gpu_matches_reference_fixture(name, precision):
    import os
    g = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", f"{name}.npz")))
    spec = eval(str(g["spec"]))
    p = pb.Problem(*spec).build()
    got = p.contract_groups(g["group_fixed"], precision=precision)
    for i in range(len(g["group_fixed"])):
        assert rel(got[i], g["amplitudes"][i]) < TOL[precision], (name, i)


# ---- full-size (BASELINE cfg2 circuit, n = 30) -------------------------------
def test_cfg2_circuit_pair_matches_live_reference(ref):
    """One (group, slice) of the 30-qubit cfg2 circuit, planned at 2^27 B so the
    reference executor finishes in seconds; GPU f64 and tf32 vs the reference."""
    spec = (30, 14, "grid(5,6)", 1, list(range(6)), 1 << 27, "low")
    r = ref.RefProblem(*spec).build()
    p = pb.Problem(*spec).build()
    assert np.array_equal(r.plan["steps"], p.plan["steps"])
    fixed, _ = pb.build_candidate_set(30, list(range(6)), 2, pb.split_next(1, 0xCA11D))
    want = r.execute_gsc(int(fixed[0]), 3)
    for precision in ("f64", "tf32", "bf16", "f16"):
        got = p.contract_groups(fixed[:1], precision=precision, configs=None, slices=(3, 4))[0]
        print(precision, rel(got, want))
        assert rel(got, want) < TOL[precision], precision


def test_cfg2_full_size_properties():
    """BASELINE cfg2 plan (2^8 slices): slice-range linearity, group batching vs
    single groups, tf32 vs f64 on the same slices."""
    p = pb.Problem(30, 14, "grid(5,6)", 1, list(range(6)), 3 << 30, "low").build()
    fixed, _ = pb.build_candidate_set(30, list(range(6)), 8, pb.split_next(1, 0xCA11D))
    both = p.contract_groups(fixed, precision="tf32", configs=None, slices=(0, 2))
    s0 = p.contract_groups(fixed, precision="tf32", configs=None, slices=(0, 1))
    s1 = p.contract_groups(fixed, precision="tf32", configs=None, slices=(1, 2))
    assert rel(s0 + s1, both) < 1e-6
    # a different batch changes GEMM shapes (M fold, split-K), hence tf32 rounding
    single = p.contract_groups(fixed[3:4], precision="tf32", configs=None, slices=(0, 2))[0]
    assert rel(single, both[3]) < 1e-3
    # the same call is deterministic bit for bit (fixed-order reductions, no float atomics)
    again = p.contract_groups(fixed, precision="tf32", configs=None, slices=(0, 2))
    assert np.array_equal(again, both)
    exact = p.contract_groups(fixed[:2], precision="f64", configs=None, slices=(0, 2))
    for g in range(2):
        assert rel(both[g], exact[g]) < TOL["tf32"]


@pytest.mark.parametrize("precision", ["f64", "tf32", "f16"])
def test_sycamore53_sliced_matches_oracle(precision):
    """Sycamore-53 layout (configs 3-4 topology) at m = 6, sliced to 2^7 slices by a
    2^20 B budget: GPU groups vs the C restatement, plus slice-range linearity."""
    p = pb.Problem(53, 6, "sycamore53", 1, list(range(6)), 1 << 20, "low").build()
    assert p.n_slices == 128
    pn = port.PortNet(p.net, p.plan)
    fixed, _ = pb.build_candidate_set(53, list(range(6)), 4, pb.split_next(1, 0xCA11D))
    got = p.contract_groups(fixed[:2], precision=precision)
    for g in range(2):
        assert rel(got[g], pn.contract_group(int(fixed[g]))) < TOL[precision], (g, precision)
    a = p.contract_groups(fixed[:2], precision=precision, configs=None, slices=(0, 40))
    b = p.contract_groups(fixed[:2], precision=precision, configs=None, slices=(40, 128))
    assert rel(a + b, got) < (1e-12 if precision == "f64" else TOL[precision])


def test_scheduler_blocks_on_gpu_equal_single_call():
    from paper_2406_18889_b200 import scheduler
    p = pb.Problem(10, 10, "line", 17, [0, 3, 5, 8], 20000, "low").build()
    fixed = np.array([0, 5, 22, 63], np.uint64)
    full = p.contract_groups(fixed, precision="f64", configs=None)
    got = scheduler.contract_sharded(scheduler.gpu_block_fn(p, fixed, "f64"), p.n_slices)
    assert got.is_cuda
    assert rel(got.cpu().numpy(), full) < 1e-12


# ---- batch-aware reassociation, level-0 caching, async calls ------------------
def test_reassociated_tree_matches_plan_tree(monkeypatch):
    """The executor reassociates the plan's tree for the group batch (rotations
    that keep every node's subtree); amplitudes equal the plan-tree execution
    to rounding, and the executed FLOPs drop."""
    spec = (30, 14, "grid(5,6)", 1, list(range(6)), 3 << 30, "low")
    fixed, _ = pb.build_candidate_set(30, list(range(6)), 8, pb.split_next(1, 0xCA11D))
    from paper_2406_18889_b200._native import rcsg_stats
    st_r, st_p = rcsg_stats(), rcsg_stats()
    got = pb.Problem(*spec).build().contract_groups(fixed, precision="f64", configs=None, slices=(5, 6), stats=st_r)
    monkeypatch.setenv("RCSG_TREE", "plan")
    want = pb.Problem(*spec).build().contract_groups(fixed, precision="f64", configs=None, slices=(5, 6),
                                                     stats=st_p)
    for g in range(len(fixed)):
        assert rel(got[g], want[g]) < 1e-12, g
    assert st_r.executed_flops * 4 < st_p.executed_flops, (st_r.executed_flops, st_p.executed_flops)
    assert st_r.plan_flops == st_p.plan_flops  # reference-equivalent work is the plan's


def test_level0_cache_across_calls_and_async():
    """Level-0 results are computed once and reused by later calls; async calls
    accumulate the same sums as synchronous ones."""
    import torch
    p = pb.Problem(10, 10, "line", 17, [0, 3, 5, 8], 20000, "low").build()
    fixed = np.array([0, 5, 22, 63], np.uint64)
    full = p.contract_groups(fixed, precision="f64", configs=None)
    acc = torch.zeros(len(fixed) * 16 * 2, dtype=torch.float64, device="cuda")
    for s in range(p.n_slices):
        p.contract_groups_device(fixed, acc.data_ptr(), precision="f64", configs=None, slices=(s, s + 1),
                                 sync=False)
    p.sync("f64")
    got = acc.cpu().numpy().view(np.complex128).reshape(len(fixed), -1)
    assert rel(got, full) < 1e-12


def test_async_numeric_fault_is_deferred_to_sync():
    import torch
    inf = float("inf")
    p = pb.Problem.from_network([2, 1], [0, 1, 1], [inf, 0, 0, 1, 1, 1], ["a", "b"], 1, [0], [0], [0])
    acc = torch.zeros(4, dtype=torch.float64, device="cuda")
    p.contract_groups_device([0], acc.data_ptr(), precision="f64", configs=None, sync=False)
    with pytest.raises(pb.NumericFault):
        p.sync("f64")


@pytest.mark.parametrize("precision", ["f64", "f16"])
def test_slice_tables_match_per_pass_evaluation(monkeypatch, precision):
    """Small per-pass subtrees are tabulated over their sliced labels once per
    binding and gathered each pass; the amplitudes equal the per-pass
    evaluation bit for bit (same kernels on the same data, evaluated earlier)."""
    spec = (30, 14, "grid(5,6)", 1, list(range(6)), 3 << 30, "low")
    fixed, _ = pb.build_candidate_set(30, list(range(6)), 8, pb.split_next(1, 0xCA11D))
    tab = pb.Problem(*spec).build().contract_groups(fixed, precision=precision, configs=None, slices=(37, 41))
    monkeypatch.setenv("RCSG_NO_TABLES", "1")
    ref = pb.Problem(*spec).build().contract_groups(fixed, precision=precision, configs=None, slices=(37, 41))
    assert np.array_equal(tab, ref)


def test_slice_tables_on_sliced_line_against_oracle():
    p = pb.Problem(10, 10, "line", 17, [0, 3, 5, 8], 20000, "low").build()
    pn = port.PortNet(p.net, p.plan)
    fixed = np.array([0, 5, 22, 63], np.uint64)
    got = p.contract_groups(fixed, precision="f64", configs=None)
    for g, fb in enumerate(fixed):
        assert rel(got[g], pn.contract_group(int(fb))) < 1e-10


def test_group_chunks_under_a_tight_memory_budget():
    """A memory budget below the one-chunk arena splits the groups into chunks
    (group-only subtrees then run inside every pass, per chunk); the amplitudes
    equal the single-chunk run up to f64 summation order (chunk-sized GEMM
    shapes change the split-K choices)."""
    from paper_2406_18889_b200._native import rcsg_stats
    spec = (30, 14, "grid(5,6)", 1, list(range(6)), 3 << 30, "low")
    fixed, _ = pb.build_candidate_set(30, list(range(6)), 256, pb.split_next(1, 0xCA11D))
    st0, st1, st2 = rcsg_stats(), rcsg_stats(), rcsg_stats()
    pb.Problem(*spec).build().contract_groups(fixed[:1], precision="f64", configs=None, slices=(3, 4), stats=st0)
    one = pb.Problem(*spec).build().contract_groups(fixed, precision="f64", configs=None, slices=(3, 5), stats=st1)
    tight = int(st0.arena_bytes + (st1.arena_bytes - st0.arena_bytes) / 3)  # ~3 chunks
    many = pb.Problem(*spec).build().contract_groups(fixed, precision="f64", configs=None, slices=(3, 5),
                                                     budget=tight, stats=st2)
    assert st2.arena_bytes < st1.arena_bytes
    assert st2.passes > st1.passes  # passes count (config, slice, chunk) triples
    for g in range(len(fixed)):
        assert rel(many[g], one[g]) < 1e-12, g


def test_f16_overflow_widens_scales_and_retries(monkeypatch):
    """fp16 scales 2^12 too tight (RCSG_F16_BIAS=-12) overflow on the first try;
    a synchronous call then widens the headroom and reruns, and the amplitudes
    still meet the fp16 tolerance against the oracle."""
    monkeypatch.setenv("RCSG_F16_BIAS", "-12")
    p, fixed = cfg1(32)
    pn = port.PortNet(p.net, p.plan)
    got = p.contract_groups(fixed, precision="f16")
    for g, fb in enumerate(fixed):
        assert rel(got[g], pn.contract_group(int(fb))) < TOL["f16"], g


@pytest.mark.parametrize("precision", ["f64", "tf32", "f16"])
def test_forced_permutes_match_oracle(monkeypatch, precision):
    """RCSG_FORCE_PERMUTE=1: every step writes its natural [rows | cols] order and
    the consumers transpose with the bit-permutation kernel (permute.cu, the
    executor's fallback when a producer cannot write the consumer's layout);
    the amplitudes still match the oracle."""
    from paper_2406_18889_b200._native import rcsg_stats
    monkeypatch.setenv("RCSG_FORCE_PERMUTE", "1")
    p, fixed = cfg1(32)
    pn = port.PortNet(p.net, p.plan)
    p.set_profile(True)
    st = rcsg_stats()
    got = p.contract_groups(fixed, precision=precision, stats=st)
    assert st.permute_bytes > 0
    for g, fb in enumerate(fixed):
        assert rel(got[g], pn.contract_group(int(fb))) < TOL[precision], g


# ---- the bench's own headline configuration, pinned ---------------------------
def test_headline_bench_configuration_pinned(ref):
    """bench.py's workload exactly: cfg2 planned at 3*2^30 B (2^8 slices), M = 1024
    groups from Rng(1).split(0xca11d), all 256 slices through the device
    accumulator, at f16 and tf32 (the timed modes) and f64:
      - every group within the mode's tolerance of the GPU f64 run;
      - amplitude fidelity over all 65,536 candidates >= 1 - 1e-4 against the GPU
        statevector (bit-identical to the reference's simulate_exact);
      - 4 (group, slice) pairs of this same plan against the live reference
        executor (execute_assignment, ~2 min on the host cores)."""
    import concurrent.futures as cf
    import torch
    spec = (30, 14, "grid(5,6)", 1, list(range(6)), 3 << 30, "low")
    p = pb.Problem(*spec).build()
    r = ref.RefProblem(*spec).build()
    assert p.n_slices == 256 and np.array_equal(r.plan["steps"], p.plan["steps"])
    M, P = 1024, 64
    fixed, _ = pb.build_candidate_set(30, list(range(6)), M, pb.split_next(1, 0xCA11D))
    rfixed, _ = ref.candidates(30, list(range(6)), M, ref.split_next(1, 0xCA11D))
    assert np.array_equal(fixed, rfixed)
    pairs = [(0, 0), (0, 171), (700, 85), (700, 255)]
    with cf.ThreadPoolExecutor(2) as ex:  # the reference executor runs on the host meanwhile
        futs = {g: ex.submit(r.slices_mt, int(fixed[g]), [s for gg, s in pairs if gg == g], 2)
                for g in sorted({g for g, _ in pairs})}
        out = {}
        for prec in ("f64", "tf32", "f16"):
            acc = torch.zeros(M * P * 2, dtype=torch.float64, device="cuda")
            for s0 in range(0, 256, 8):
                p.contract_groups_device(fixed, acc.data_ptr(), precision=prec, configs=None,
                                         slices=(s0, s0 + 8), sync=False)
            p.sync(prec)
            out[prec] = acc.cpu().numpy().view(np.complex128).reshape(M, P)
        state = torch.empty(1 << 30, dtype=torch.complex128, device="cuda")
        p.exact_state_device(state.data_ptr())
        cand = np.array([pb.member(30, list(range(6)), int(f), i) for f in fixed for i in range(P)], np.int64)
        exact = state[torch.as_tensor(cand, device="cuda")].cpu().numpy().reshape(M, P)
        del state
        torch.cuda.empty_cache()
        for prec in ("f64", "tf32", "f16"):
            a = out[prec]
            fid = abs(np.vdot(exact, a)) ** 2 / (np.vdot(a, a).real * np.vdot(exact, exact).real)
            assert fid >= (1 - 1e-12 if prec == "f64" else 1 - 1e-4), (prec, fid)
            if prec != "f64":
                errs = [rel(a[g], out["f64"][g]) for g in range(M)]
                assert max(errs) < TOL[prec], (prec, max(errs))
        assert rel(out["f64"], exact) < 1e-10
        for g, fut in futs.items():
            ss = [s for gg, s in pairs if gg == g]
            want, _ = fut.result()
            for j, s in enumerate(ss):
                for prec in ("f64", "tf32", "f16"):
                    got = p.contract_groups(fixed[g:g + 1], precision=prec, configs=None, slices=(s, s + 1))[0]
                    assert rel(got, want[j]) < TOL[prec], (g, s, prec, rel(got, want[j]))


# ---- the scale planner's plans on both executors -------------------------------
def test_scale_planner_plan_on_reference_executor(ref):
    """A 54-qubit grid(6,9) m = 10 circuit planned by the scale planner (the
    reference planner's uint64 costs overflow at this size), imported
    into the reference executor (refo_set_plan): GPU amplitudes of (group, slice)
    pairs equal the reference's execute_assignment of the same plan."""
    spec = (54, 10, "grid(6,9)", 1, list(range(6)), 1 << 27, "low")
    p = pb.Problem(*spec).build(planner="scale", n_groups=1, trials=64)
    assert len(p.plan["sliced"]) >= 1
    r = ref.RefProblem(54, 10, "grid(6,9)", 1, list(range(6)), 1 << 62, "low").build()
    assert r.net["n_labels"] == p.net["n_labels"] and r.net["label_names"] == p.net["label_names"]
    r.set_plan(p.plan["steps"], p.plan["sliced"])
    fixed, _ = pb.build_candidate_set(54, list(range(6)), 4, pb.split_next(1, 0xCA11D))
    for g, s in ((0, 0), (3, p.n_slices - 1)):
        want = r.execute_gsc(int(fixed[g]), s)
        for prec in ("f64", "tf32", "f16"):
            got = p.contract_groups(fixed[g:g + 1], precision=prec, configs=None, slices=(s, s + 1))[0]
            assert rel(got, want) < TOL[prec], (g, s, prec, rel(got, want))


@pytest.mark.parametrize("precision", ["f64", "tf32"])
def test_scale_planner_sycamore_matches_oracle(precision):
    """Sycamore-53 m = 8 planned by the scale planner for a 16-group batch: GPU
    group amplitudes over two slices equal the C restatement's execution of the
    same plan."""
    p = pb.Problem(53, 8, "sycamore53", 1, list(range(6)), 1 << 26, "low").build(planner="scale", n_groups=16,
                                                                               trials=64)
    pn = port.PortNet(p.net, p.plan)
    fixed, _ = pb.build_candidate_set(53, list(range(6)), 16, pb.split_next(1, 0xCA11D))
    got = p.contract_groups(fixed, precision=precision, configs=None, slices=(0, 2))
    for g in (0, 7, 15):
        want = pn.contract_group(int(fixed[g]), slices=(0, 2))
        assert rel(got[g], want) < TOL[precision], (g, rel(got[g], want))


def test_shared_operand_variant_order_is_bit_identical(monkeypatch, capfd):
    """Batched steps whose larger operand has fewer variants than the result run
    their tiles in an order grouped by that operand's variant (tcgen05 raster
    with a variant permutation); the amplitudes are bit-identical to the plain
    order (RCSG_NO_VPERM).  cfg3's committed plan at M = 64 has such steps."""
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = pb.Problem(53, 12, "sycamore53", 1, list(range(6)), 1 << 36, "low").build(
        plan_json=open(os.path.join(root, "plans", "cfg3.json")).read())
    fixed, _ = pb.build_candidate_set(53, list(range(6)), 64, pb.split_next(1, 0xCA11D))
    monkeypatch.setenv("RCSG_DEBUG_VPERM", "1")
    a = p.contract_groups(fixed, precision="tf32", configs=None, slices=(0, 1))
    assert "[rcsg] vperm step" in capfd.readouterr().err
    p.release()
    monkeypatch.setenv("RCSG_NO_VPERM", "1")
    b = p.contract_groups(fixed, precision="tf32", configs=None, slices=(0, 1))
    p.release()
    assert np.isfinite(a).all() and np.array_equal(a, b)
