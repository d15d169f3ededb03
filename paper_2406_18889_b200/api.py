"""Python mirror of the reference's hot-path API (namespace ``rcs``), over the C ABI.

Names, argument meaning and errors follow the reference
(/root/reference/proj/include/rcs/{contraction_engine,sampling}.hpp):
``contract``, ``contract_group``, ``execute_assignment``, ``build_candidate_set``,
``top_k_select``, ``direct_sample``, ``xeb``; ``ConfigError`` / ``NumericFault`` /
``CapacityError`` carry the reference's exit codes 2 / 3 / 4.  The pipeline
inputs (circuit, network, plan) are built by the library's C++ host code,
which reproduces the reference planner bit for bit.  Every contraction and
selection runs on the GPU; nothing here computes amplitudes on the CPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native
from ._native import (PRECISIONS, rcsg_candidates, rcsg_network_desc, rcsg_plan_desc,
                      rcsg_stats)


class Error(RuntimeError):
    exit_code = 1

    def __init__(self, msg: str):
        super().__init__(msg)
        self.msg = msg


class ConfigError(Error):
    exit_code = 2


class NumericFault(Error):
    exit_code = 3

    def __init__(self, msg: str, step_index: int):
        super().__init__(msg)
        self.step_index = step_index


class CapacityError(Error):
    exit_code = 4


class DeviceError(Error):
    exit_code = 5


def _raise(rc: int, msg: str, step: int):
    if rc == _native.RCSG_ERR_CONFIG:
        raise ConfigError(msg)
    if rc == _native.RCSG_ERR_NUMERIC:
        raise NumericFault(msg, step)
    if rc == _native.RCSG_ERR_CAPACITY:
        raise CapacityError(msg)
    raise DeviceError(msg)


def _check_h(rc: int):
    if rc:
        step = C.c_int(-1)
        msg = _native.lib().rcsh_last_error(C.byref(step)).decode()
        _raise(rc, msg, step.value)


def _check_g(rc: int):
    if rc:
        step = C.c_int32(-1)
        msg = _native.lib().rcsg_last_error(C.byref(step)).decode()
        _raise(rc, msg, step.value)


def _p(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _i32(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.int32))


def _u64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.uint64))


EFFORT = {"low": 0, "medium": 1, "high": 2}


def _order_after_torch(stream_ptr: int):
    """Make the program's (non-blocking) stream wait for torch's current stream,
    so a device accumulator zeroed or written by torch is ready before the
    executor's += lands on it."""
    import sys
    torch = sys.modules.get("torch")
    if torch is None or not torch.cuda.is_available() or not stream_ptr:
        return
    cur = torch.cuda.current_stream()
    if cur.cuda_stream == stream_ptr:
        return
    ev = torch.cuda.Event()
    ev.record(cur)
    torch.cuda.ExternalStream(stream_ptr).wait_event(ev)


def _prec(p) -> int:
    if isinstance(p, str):
        if p not in PRECISIONS:
            raise ConfigError("precision must be f64, f32, tf32, 3xtf32, bf16 or f16")
        return PRECISIONS[p]
    return int(p)


@dataclass
class Problem:
    """circuit -> network(open) -> broken edges -> plan -> configs, built by the C++ host code.

    Mirrors the reference pipeline used by contract_group callers
    (harness.cpp:131-152 with open = the group's open qubits).
    """

    n: int
    cycles: int
    topology: str
    seed: int
    open: list
    budget: int
    effort: str = "low"
    k_broken: int = 0
    m: int = 1
    handle: int = 0
    net: dict = field(default_factory=dict)
    plan: dict = field(default_factory=dict)

    def build(self, planner: str | None = None, n_groups: int = 1, trials: int = 0, threads: int = 0,
              plan_json: str | None = None):
        """planner None: find_contraction_path as configured (Auto: the reference
        algorithm where it works, the scale planner where it overflows);
        "reference" / "scale" / "auto" select explicitly.  n_groups, trials and
        threads tune the scale planner; its report lands in self.plan_report.
        plan_json: skip planning and import this plan.json instead."""
        if plan_json is not None:
            planner = "none"
        h = C.c_void_p()
        op = _i32(self.open)
        if planner is None:
            _check_h(_native.lib().rcsh_build(self.n, self.cycles, self.topology.encode(),
                                              C.c_uint64(self.seed), _p(op, C.c_int), len(self.open),
                                              C.c_uint64(self.budget), EFFORT[self.effort], self.k_broken,
                                              C.c_uint64(self.m), C.byref(h)))
            self.plan_report = None
        else:
            rep = np.zeros(10, np.float64)
            kind = {"reference": 0, "scale": 1, "auto": 2, "none": 3}[planner]
            _check_h(_native.lib().rcsh_build_ex(self.n, self.cycles, self.topology.encode(),
                                                 C.c_uint64(self.seed), _p(op, C.c_int), len(self.open),
                                                 C.c_uint64(self.budget), EFFORT[self.effort], self.k_broken,
                                                 C.c_uint64(self.m), kind, C.c_uint64(n_groups), trials, threads,
                                                 _p(rep, C.c_double), C.byref(h)))
            keys = ["log2_total_flops", "log2_flops_per_slice_batched", "log2_flops_once_batched",
                    "log2_max_size", "seconds", "n_sliced", "trials", "winning_trial", "threads",
                    "reduced_tensors"]
            self.plan_report = dict(zip(keys, rep.tolist())) if rep[0] != -1.0 else None
        self.handle = h
        if plan_json is not None:
            return self.import_plan(plan_json)
        self._export()
        return self

    @classmethod
    def from_network(cls, leaf_rank, leaf_labels, leaf_data, names, n_qubits, output_labels,
                     open_labels, open_qubits, budget=1 << 30, effort="medium", seed=0, broken=()):
        """find_contraction_path over a hand-built TensorNetwork (tensor_network.hpp:26-43)."""
        self = cls(n=n_qubits, cycles=0, topology="custom", seed=seed, open=list(open_qubits),
                   budget=budget, effort=effort)
        h = C.c_void_p()
        rk, lb = _i32(leaf_rank), _i32(leaf_labels)
        data = np.ascontiguousarray(np.asarray(leaf_data, np.complex128)).view(np.float64)
        ol, opl, opq, br = _i32(output_labels), _i32(open_labels or [0]), _i32(open_qubits or [0]), _i32(list(broken) or [0])
        _check_h(_native.lib().rcsh_build_network(
            len(rk), _p(rk, C.c_int), _p(lb, C.c_int), _p(data, C.c_double), "\n".join(names).encode(),
            n_qubits, _p(ol, C.c_int), len(open_labels), _p(opl, C.c_int), _p(opq, C.c_int),
            C.c_uint64(budget), EFFORT[effort], C.c_uint64(seed), len(broken), _p(br, C.c_int),
            C.byref(h)))
        self.handle = h
        self._export()
        return self

    def __del__(self):
        if self.handle and _native._lib is not None:
            _native._lib.rcsh_free(self.handle)
            self.handle = 0

    def _export(self):
        L = _native.lib()
        sz = np.zeros(8, np.int64)
        L.rcsh_net_sizes(self.handle, _p(sz, C.c_int64))
        n_leaves, n_labels, n_q, n_open, sum_rank, sum_amps, n_layers, n_edges = map(int, sz)
        rank = np.zeros(n_leaves, np.int32)
        labels = np.zeros(max(sum_rank, 1), np.int32)
        data = np.zeros(2 * sum_amps, np.float64)
        out_l = np.zeros(max(n_q, 1), np.int32)
        open_l = np.zeros(max(n_open, 1), np.int32)
        open_q = np.zeros(max(n_open, 1), np.int32)
        L.rcsh_net_export(self.handle, _p(rank, C.c_int), _p(labels, C.c_int), _p(data, C.c_double),
                          _p(out_l, C.c_int), _p(open_l, C.c_int), _p(open_q, C.c_int))
        nbytes = L.rcsh_label_names(self.handle, None, 0)
        buf = C.create_string_buffer(int(nbytes) + 1)
        L.rcsh_label_names(self.handle, buf, nbytes + 1)
        names = buf.value.decode().split("\n")[:-1]
        edges = np.zeros(3 * max(n_edges, 1), np.int32)
        L.rcsh_wire_edges(self.handle, _p(edges, C.c_int))
        self.net = dict(leaf_rank=rank, leaf_labels=labels[:sum_rank], leaf_data=data,
                        n_labels=n_labels, n_qubits=n_q, output_labels=out_l[:n_q],
                        open_labels=open_l[:n_open], open_qubits=open_q[:n_open], label_names=names,
                        n_layers=n_layers, wire_edges=edges[:3 * n_edges].reshape(-1, 3))
        ps = np.zeros(5, np.int64)
        L.rcsh_plan_sizes(self.handle, _p(ps, C.c_int64))
        n_steps, n_sl, n_br, n_fx, n_cfg = map(int, ps)
        steps = np.zeros((max(n_steps, 1), 6), np.int64)
        sl = np.zeros(max(n_sl, 1), np.int32)
        br = np.zeros(max(n_br, 1), np.int32)
        fx = np.zeros(max(n_fx, 1), np.int32)
        cf = np.zeros(max(n_cfg, 1), np.uint64)
        tot = np.zeros(4, np.uint64)
        L.rcsh_plan_export(self.handle, _p(steps, C.c_int64), _p(sl, C.c_int), _p(br, C.c_int),
                           _p(fx, C.c_int), _p(cf, C.c_uint64), _p(tot, C.c_uint64))
        self.plan = dict(steps=steps[:n_steps], sliced=sl[:n_sl], broken=br[:n_br],
                         fixed_outputs=fx[:n_fx], configs=cf[:n_cfg],
                         flops_per_slice=int(tot[0]), traffic_bytes_per_slice=int(tot[1]),
                         peak_bytes=int(tot[2]), memory_budget_bytes=int(tot[3]))

    def plan_json(self) -> str:
        """plan_to_json (contraction_plan.cpp:451-491), byte-identical to the reference's."""
        n = _native.lib().rcsh_plan_json(self.handle, None, 0)
        buf = C.create_string_buffer(int(n) + 1)
        _native.lib().rcsh_plan_json(self.handle, buf, n + 1)
        return buf.value.decode()

    def import_plan(self, text: str):
        """Replace the plan with one read from plan.json (the reference's or ours)."""
        _check_h(_native.lib().rcsh_plan_import(self.handle, text.encode()))
        self._export()
        return self

    def stream(self, precision="tf32", budget=0) -> int:
        """cudaStream_t (as int) the compiled program launches on."""
        out = C.c_void_p()
        _check_h(_native.lib().rcsh_program_stream(self.handle, _prec(precision), C.c_uint64(budget),
                                                   C.byref(out)))
        return out.value or 0

    def release(self):
        """Free the compiled device programs (and their arenas) of this problem."""
        _native.lib().rcsh_release_programs(self.handle)

    def set_profile(self, on: bool):
        """Per-kernel-class CUDA-event timing into rcsg_stats (gemm_ms, permute_ms, ...)."""
        _native.lib().rcsh_set_profile(self.handle, 1 if on else 0)

    @property
    def n_open(self) -> int:
        return len(self.net["open_labels"])

    @property
    def n_slices(self) -> int:
        return 1 << len(self.plan["sliced"])

    def gates(self) -> np.ndarray:
        n = _native.lib().rcsh_circuit_gates(self.handle, None)
        out = np.zeros(4 * max(n, 1), np.int32)
        _native.lib().rcsh_circuit_gates(self.handle, _p(out, C.c_int))
        return out[:4 * n].reshape(-1, 4)

    # ---- exact oracle -------------------------------------
    def exact_state_device(self, d_state: int):
        """simulate_exact (statevector.cpp:79-86) into a DEVICE buffer of 2^n
        interleaved complex f64 (e.g. a torch.complex128 tensor's data_ptr())."""
        _check_h(_native.lib().rcsh_statevector(self.handle, C.c_void_p(d_state)))

    def exact_probabilities(self, indices) -> np.ndarray:
        """Ideal probabilities |<x|C|0>|^2 of the given basis indices (qubit q =
        bit q), from the GPU statevector (n <= 33 fits one B200)."""
        import torch
        state = torch.empty(1 << self.n, dtype=torch.complex128, device="cuda")
        self.exact_state_device(state.data_ptr())
        idx = _u64(indices)
        out = np.zeros(len(idx), np.float64)
        _check_g(_native.lib().rcsg_statevector_probs(C.c_void_p(state.data_ptr()), C.c_uint64(len(idx)),
                                                    _p(idx, C.c_uint64), _p(out, C.c_double)))
        del state
        return out

    # ---- hot path ---------------------------------------------------------
    def contract_groups(self, fixed, precision="f64", configs="all", slices=None, budget=0,
                        stats: rcsg_stats | None = None) -> np.ndarray:
        """Amplitudes [G][2^l] of every group (rcsg_contract_groups).

        configs: "all" -> the plan's BrokenEdgeConfig; None -> exact; list -> those bits.
        slices: (begin, end) slice range, default all.
        """
        fixed = _u64(fixed)
        s0, s1 = slices if slices is not None else (0, self.n_slices)
        if isinstance(configs, str):
            n_cfg, cf = -1, _u64([0])
        elif configs is None:
            n_cfg, cf = 0, _u64([0])
        else:
            cf = _u64(configs)
            n_cfg = len(cf)
        out = np.zeros(2 * (len(fixed) << self.n_open), np.float64)
        st = stats if stats is not None else rcsg_stats()
        _check_h(_native.lib().rcsh_contract_groups(
            self.handle, _prec(precision), C.c_uint64(budget), C.c_uint64(len(fixed)),
            _p(fixed, C.c_uint64), n_cfg, _p(cf, C.c_uint64), C.c_uint64(s0), C.c_uint64(s1),
            _p(out, C.c_double), C.byref(st)))
        return out.view(np.complex128).reshape(len(fixed), -1)

    def contract_groups_device(self, fixed, d_acc: int, precision="tf32", configs="all",
                               slices=None, budget=0, stats: rcsg_stats | None = None, sync=True):
        """Accumulate into a DEVICE float64 buffer (e.g. a torch tensor's data_ptr()).

        sync=False returns once the work is enqueued on the program's stream
        (self.stream(precision)); a NumericFault is then raised by the next
        synchronous call or by self.sync(precision)."""
        fixed = _u64(fixed)
        s0, s1 = slices if slices is not None else (0, self.n_slices)
        if isinstance(configs, str):
            n_cfg, cf = -1, _u64([0])
        elif configs is None:
            n_cfg, cf = 0, _u64([0])
        else:
            cf = _u64(configs)
            n_cfg = len(cf)
        st = stats if stats is not None else rcsg_stats()
        _order_after_torch(self.stream(precision, budget))
        _check_h(_native.lib().rcsh_contract_groups_device(
            self.handle, _prec(precision), C.c_uint64(budget), C.c_uint64(len(fixed)),
            _p(fixed, C.c_uint64), n_cfg, _p(cf, C.c_uint64), C.c_uint64(s0), C.c_uint64(s1),
            C.c_void_p(d_acc), C.byref(st), int(bool(sync))))
        return st

    def sync(self, precision="tf32", budget=0):
        """Wait for the program's stream; raises a deferred NumericFault."""
        _check_h(_native.lib().rcsh_program_sync(self.handle, _prec(precision), C.c_uint64(budget)))

    def contract_group(self, fixed_bits: int, precision="f64") -> np.ndarray:
        """contract_group (contraction_engine.cpp:307-325)."""
        return self.contract_groups([fixed_bits], precision=precision)[0]

    def contract(self, fixed: dict | None = None, configs=None, precision="f64"):
        """contract (contraction_engine.cpp:210-305) -> (amplitudes, flops)."""
        fixed = fixed or {}
        fl = _i32(list(fixed.keys()) or [0])
        fv = _i32(list(fixed.values()) or [0])
        n_cfg = 0 if configs is None else (-1 if isinstance(configs, str) else len(configs))
        cf = _u64([0] if configs is None or isinstance(configs, str) else configs)
        n_free = sum(1 for l in self.net["open_labels"] if int(l) not in fixed)
        out = np.zeros(2 << n_free, np.float64)
        flops = C.c_uint64()
        _check_h(_native.lib().rcsh_contract(self.handle, _prec(precision), len(fixed), _p(fl, C.c_int),
                                             _p(fv, C.c_int), n_cfg, _p(cf, C.c_uint64),
                                             _p(out, C.c_double), C.byref(flops)))
        return out.view(np.complex128), flops.value

    def execute(self, assignment: dict, precision="f64") -> np.ndarray:
        """execute_assignment (contraction_engine.cpp:153-208)."""
        ls = _i32(list(assignment.keys()) or [0])
        vs = _i32(list(assignment.values()) or [0])
        n = C.c_int64()
        _check_h(_native.lib().rcsh_execute(self.handle, _prec(precision), len(assignment),
                                            _p(ls, C.c_int), _p(vs, C.c_int), None, C.byref(n)))
        out = np.zeros(2 * n.value, np.float64)
        _check_h(_native.lib().rcsh_execute(self.handle, _prec(precision), len(assignment),
                                            _p(ls, C.c_int), _p(vs, C.c_int), _p(out, C.c_double),
                                            C.byref(n)))
        return out.view(np.complex128)

    def assignment_gsc(self, fixed_bits: int, slice_idx: int, config_bits: int = 0) -> dict:
        """The assignment contract()/contract_group() build for (group, slice, config)
        (contraction_engine.cpp:242-248, 310-318)."""
        a = {}
        open_q = set(int(q) for q in self.net["open_qubits"])
        b = 0
        for q in range(self.net["n_qubits"]):
            if q in open_q:
                continue
            a[int(self.net["output_labels"][q])] = (fixed_bits >> b) & 1
            b += 1
        for i, l in enumerate(self.plan["broken"]):
            a[int(l)] = (config_bits >> i) & 1
        for i, l in enumerate(self.plan["sliced"]):
            a[int(l)] = (slice_idx >> i) & 1
        return a


# ---- descriptor-level entry (hand-built networks, KATs) --------------------
def execute_desc(net: dict, steps, assign, precision="f64") -> np.ndarray:
    """rcsg_execute_assignment on raw arrays: net = dict(leaf_rank, leaf_labels, leaf_data
    (complex), n_labels, n_qubits, output_labels, open_labels, open_qubits); steps = [(l, r, res)]."""
    rk, lb = _i32(net["leaf_rank"]), _i32(list(net["leaf_labels"]) or [0])
    data = np.ascontiguousarray(np.asarray(net["leaf_data"], np.complex128)).view(np.float64)
    ol = _i32(list(net["output_labels"]) or [0])
    opl, opq = _i32(list(net["open_labels"]) or [0]), _i32(list(net["open_qubits"]) or [0])
    st = _i32(np.asarray(steps, np.int32).reshape(-1)[:].tolist() or [0])
    nd = rcsg_network_desc(len(rk), _p(rk, C.c_int32), _p(lb, C.c_int32), _p(data, C.c_double),
                           int(net["n_labels"]), int(net["n_qubits"]), _p(ol, C.c_int32),
                           len(net["open_labels"]), _p(opl, C.c_int32), _p(opq, C.c_int32))
    z = _i32([0])
    pd = rcsg_plan_desc(len(steps), _p(st, C.c_int32), 0, _p(z, C.c_int32), 0, _p(z, C.c_int32), 0,
                        _p(z, C.c_int32))
    a = np.ascontiguousarray(np.asarray(assign, np.int8))
    n = C.c_uint64()
    _check_g(_native.lib().rcsg_execute_assignment(C.byref(nd), C.byref(pd), _prec(precision),
                                                   _p(a, C.c_int8), None, C.byref(n)))
    out = np.zeros(2 * n.value, np.float64)
    _check_g(_native.lib().rcsg_execute_assignment(C.byref(nd), C.byref(pd), _prec(precision),
                                                   _p(a, C.c_int8), _p(out, C.c_double), C.byref(n)))
    return out.view(np.complex128)


# ---- sampler ---------------------------------------------------------------
def build_candidate_set(n: int, open_qubits, n_groups: int, seed: int):
    """build_candidate_set (sampling.cpp:29-60) -> (group_fixed, duplicate_groups)."""
    op = _i32(sorted(open_qubits) or [0])
    out = np.zeros(max(n_groups, 1), np.uint64)
    dup = C.c_int()
    _check_h(_native.lib().rcsh_candidates(n, _p(op, C.c_int), len(open_qubits), C.c_uint64(n_groups),
                                           C.c_uint64(seed), _p(out, C.c_uint64), C.byref(dup)))
    return out, dup.value


def member(n: int, open_qubits, fixed: int, i: int) -> int:
    op = _i32(sorted(open_qubits) or [0])
    return int(_native.lib().rcsh_member(n, _p(op, C.c_int), len(open_qubits), C.c_uint64(fixed),
                                         C.c_uint64(i)))


def top_k_select(n, open_qubits, fixed, probs, k) -> np.ndarray:
    """top_k_select with probs [G][2^l] as the ProbFn (GPU selection)."""
    op = _i32(sorted(open_qubits) or [0])
    fixed = _u64(fixed)
    probs = np.ascontiguousarray(probs, np.float64)
    out = np.zeros(max(int(k), 1), np.uint64)
    _check_h(_native.lib().rcsh_topk(n, _p(op, C.c_int), len(open_qubits), C.c_uint64(len(fixed)),
                                     _p(fixed, C.c_uint64), _p(probs, C.c_double), C.c_uint64(k),
                                     _p(out, C.c_uint64)))
    return out[:k]


def direct_sample(n, open_qubits, fixed, probs, seed) -> np.ndarray:
    """direct_sample with probs [G][2^l] as the ProbFn (GPU sampling)."""
    op = _i32(sorted(open_qubits) or [0])
    fixed = _u64(fixed)
    probs = np.ascontiguousarray(probs, np.float64)
    out = np.zeros(len(fixed), np.uint64)
    _check_h(_native.lib().rcsh_direct(n, _p(op, C.c_int), len(open_qubits), C.c_uint64(len(fixed)),
                                       _p(fixed, C.c_uint64), _p(probs, C.c_double),
                                       C.c_uint64(seed), _p(out, C.c_uint64)))
    return out


def _cands(n, open_qubits, fixed):
    op = _i32(sorted(open_qubits) or [0])
    fx = _u64(fixed)
    cs = rcsg_candidates(n, len(open_qubits), _p(op, C.c_int32), len(fx), _p(fx, C.c_uint64))
    return cs, (op, fx)


def top_k_from_device_amps(n, open_qubits, fixed, d_amps: int, k: int) -> np.ndarray:
    """Fused |a|^2 + global top-k on DEVICE amplitudes [G][2^l] (rcsg_topk)."""
    cs, keep = _cands(n, open_qubits, fixed)
    out = np.zeros(k, np.uint64)
    _check_g(_native.lib().rcsg_topk(C.byref(cs), C.c_void_p(d_amps), C.c_uint64(k), _p(out, C.c_uint64)))
    return out


def direct_from_device_amps(n, open_qubits, fixed, d_amps: int, seed: int) -> np.ndarray:
    cs, keep = _cands(n, open_qubits, fixed)
    out = np.zeros(len(keep[1]), np.uint64)
    _check_g(_native.lib().rcsg_direct_sample(C.byref(cs), C.c_void_p(d_amps), C.c_uint64(seed),
                                              _p(out, C.c_uint64)))
    return out


def postprocess_device_amps(n, open_qubits, fixed, d_amps: int, k: int = 0, direct_seed=None,
                            d_state: int = 0):
    """Fused post-processing (rcsg_postprocess) of DEVICE amplitudes [G][2^l]:
    top-k (k > 0), one direct sample per group (direct_seed given) from the same
    streaming pass, and the XEB of both against a DEVICE statevector d_state.
    Returns (top or None, direct or None, stats dict)."""
    cs, keep = _cands(n, open_qubits, fixed)
    top = np.zeros(max(k, 1), np.uint64)
    direct = np.zeros(len(keep[1]), np.uint64)
    st = _native.rcsg_post_stats()
    _check_g(_native.lib().rcsg_postprocess(
        C.byref(cs), C.c_void_p(d_amps), C.c_uint64(k), _p(top, C.c_uint64) if k else None,
        1 if direct_seed is not None else 0, C.c_uint64(direct_seed or 0),
        _p(direct, C.c_uint64) if direct_seed is not None else None, C.c_void_p(d_state or None), C.byref(st)))
    return (top[:k] if k else None), (direct if direct_seed is not None else None), st.as_dict()


def xeb_state(n: int, samples, d_state: int) -> float:
    """xeb with ideal q read from a DEVICE statevector (rcsg_xeb_state)."""
    idx = _u64(samples)
    out = C.c_double()
    _check_g(_native.lib().rcsg_xeb_state(n, C.c_uint64(len(idx)), _p(idx, C.c_uint64), C.c_void_p(d_state),
                                          C.byref(out)))
    return out.value


def xeb(n: int, q) -> float:
    """xeb (sampling.cpp:62-73) over the ideal probabilities q of the samples."""
    q = np.ascontiguousarray(q, np.float64)
    out = C.c_double()
    _check_g(_native.lib().rcsg_xeb(n, C.c_uint64(len(q)), _p(q, C.c_double), C.byref(out)))
    return out.value


def state_fidelity(approx, exact):
    """state_fidelity (contraction_engine.cpp:327-345) -> (value, zero_norm_warning)."""
    a = np.ascontiguousarray(np.asarray(approx, np.complex128)).view(np.float64)
    e = np.ascontiguousarray(np.asarray(exact, np.complex128)).view(np.float64)
    if a.size != e.size:
        raise ConfigError("fidelity requires identical index sets")
    out, warn = C.c_double(), C.c_int()
    _check_h(_native.lib().rcsh_state_fidelity(C.c_uint64(a.size // 2), _p(a, C.c_double), _p(e, C.c_double),
                                               C.byref(out), C.byref(warn)))
    return out.value, bool(warn.value)


def predicted_topk_xeb(fidelity: float, candidate_size: int, k: int) -> float:
    """predicted_topk_xeb (sampling.cpp:147-151): F * ln(|S| / k)."""
    out = C.c_double()
    _check_h(_native.lib().rcsh_predicted_topk_xeb(C.c_double(fidelity), C.c_uint64(candidate_size),
                                                   C.c_uint64(k), C.byref(out)))
    return out.value


def timings_to_csv(ids, bits, ms, flops) -> str:
    """timings_to_csv (contraction_engine.cpp:347-354)."""
    ids, bits, flops = _u64(ids), _u64(bits), _u64(flops)
    ms = np.ascontiguousarray(ms, np.float64)
    args = (len(ids), _p(ids, C.c_uint64), _p(bits, C.c_uint64), _p(ms, C.c_double), _p(flops, C.c_uint64))
    n = _native.lib().rcsh_timings_csv(*args, None, 0)
    buf = C.create_string_buffer(int(n) + 1)
    _native.lib().rcsh_timings_csv(*args, buf, n + 1)
    return buf.value.decode()


def samples_to_text(n_qubits: int, samples, topk: bool = False, k: int = 0) -> str:
    """samples_to_text (sampling.cpp:177-191): character q = qubit q."""
    s = _u64(samples)
    args = (n_qubits, int(topk), C.c_uint64(k), C.c_int64(len(s)), _p(s, C.c_uint64))
    n = _native.lib().rcsh_samples_text(*args, None, 0)
    buf = C.create_string_buffer(int(n) + 1)
    _native.lib().rcsh_samples_text(*args, buf, n + 1)
    return buf.value.decode()


def samples_from_text(text: str):
    """samples_from_text (sampling.cpp:193-210) -> (n_qubits, topk, k, samples)."""
    meta = np.zeros(3, np.uint64)
    raw = text.encode()
    n = _native.lib().rcsh_samples_parse(raw, _p(meta, C.c_uint64), None)
    out = np.zeros(max(int(n), 1), np.uint64)
    _native.lib().rcsh_samples_parse(raw, _p(meta, C.c_uint64), _p(out, C.c_uint64))
    return int(meta[0]), bool(meta[1]), int(meta[2]), out[:n]


def split_next(seed: int, tag: int) -> int:
    """Rng(seed).split(tag).next_u64() (rng.hpp:36-41)."""
    return int(_native.lib().rcsh_rng_split_next(C.c_uint64(seed), C.c_uint64(tag)))


def lexkey(index: int, n: int) -> int:
    return int(_native.lib().rcsh_lexkey(C.c_uint64(index), n))


def broken_configs(k: int, m: int, seed: int) -> np.ndarray:
    out = np.zeros(max(m, 1), np.uint64)
    _check_h(_native.lib().rcsh_broken_configs(k, C.c_uint64(m), C.c_uint64(seed), _p(out, C.c_uint64)))
    return out[:m]


def set_device(device: int):
    _check_g(_native.lib().rcsg_set_device(device))
