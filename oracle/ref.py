"""TEST INFRASTRUCTURE ONLY — ctypes driver for the unmodified reference library.

oracle/_ref/librcs_ref.so is the reference's own src/*.cpp compiled by
oracle/Makefile plus oracle/ref_shim.cpp (our flat C ABI).  See ref_shim.cpp for
the reference call each entry point wraps.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "librcs_ref.so")

_lib = None


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str, step: int = -1):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg
        self.step = step


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle`")
        L = C.CDLL(LIB_PATH)
        L.refo_last_error.restype = C.c_char_p
        L.refo_member.restype = C.c_uint64
        L.refo_rng_split_next.restype = C.c_uint64
        L.refo_lexkey.restype = C.c_uint64
        L.refo_circuit_gates.restype = C.c_int64
        L.refo_label_names.restype = C.c_int64
        L.refo_plan_json.restype = C.c_int64
        L.refo_timings_csv.restype = C.c_int64
        L.refo_samples_text.restype = C.c_int64
        for name in ("refo_build", "refo_contract_group", "refo_contract", "refo_execute",
                     "refo_execute_gsc", "refo_exact", "refo_candidates", "refo_topk",
                     "refo_direct", "refo_xeb", "refo_groups_mt", "refo_slices_mt", "refo_set_plan"):
            getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def _check(rc: int):
    if rc:
        step = C.c_int(-1)
        msg = lib().refo_last_error(C.byref(step)).decode()
        raise RefError(rc, msg, step.value)


def _p(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _ints(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.int32))


def _u64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.uint64))


def _cplx(buf: np.ndarray) -> np.ndarray:
    return buf.view(np.complex128)


EFFORT = {"low": 0, "medium": 1, "high": 2}


@dataclass
class RefProblem:
    """One reference pipeline: circuit -> network(open) -> broken edges -> plan -> configs."""

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

    def build(self):
        h = C.c_void_p()
        op = _ints(self.open)
        _check(lib().refo_build(self.n, self.cycles, self.topology.encode(), C.c_uint64(self.seed),
                                _p(op, C.c_int), len(self.open), C.c_uint64(self.budget),
                                EFFORT[self.effort], self.k_broken, C.c_uint64(self.m),
                                C.byref(h)))
        self.handle = h
        self._export()
        return self

    def __del__(self):
        if self.handle and _lib is not None:
            _lib.refo_free(self.handle)
            self.handle = 0

    def _export(self):
        L = lib()
        sz = np.zeros(8, np.int64)
        L.refo_net_sizes(self.handle, _p(sz, C.c_int64))
        n_leaves, n_labels, n_q, n_open, sum_rank, sum_amps, n_layers, n_edges = map(int, sz)
        rank = np.zeros(n_leaves, np.int32)
        labels = np.zeros(sum_rank, np.int32)
        data = np.zeros(2 * sum_amps, np.float64)
        out_l = np.zeros(n_q, np.int32)
        open_l = np.zeros(max(n_open, 1), np.int32)
        open_q = np.zeros(max(n_open, 1), np.int32)
        L.refo_net_export(self.handle, _p(rank, C.c_int), _p(labels, C.c_int), _p(data, C.c_double),
                          _p(out_l, C.c_int), _p(open_l, C.c_int), _p(open_q, C.c_int))
        nbytes = L.refo_label_names(self.handle, None, 0)
        buf = C.create_string_buffer(int(nbytes) + 1)
        L.refo_label_names(self.handle, buf, nbytes + 1)
        names = buf.value.decode().split("\n")[:-1]
        edges = np.zeros(3 * max(n_edges, 1), np.int32)
        L.refo_wire_edges(self.handle, _p(edges, C.c_int))
        self.net = dict(leaf_rank=rank, leaf_labels=labels, leaf_data=data, n_labels=n_labels,
                        n_qubits=n_q, output_labels=out_l, open_labels=open_l[:n_open],
                        open_qubits=open_q[:n_open], label_names=names, n_layers=n_layers,
                        wire_edges=edges[:3 * n_edges].reshape(-1, 3))
        ps = np.zeros(5, np.int64)
        L.refo_plan_sizes(self.handle, _p(ps, C.c_int64))
        n_steps, n_sl, n_br, n_fx, n_cfg = map(int, ps)
        steps = np.zeros((max(n_steps, 1), 6), np.int64)
        sl = np.zeros(max(n_sl, 1), np.int32)
        br = np.zeros(max(n_br, 1), np.int32)
        fx = np.zeros(max(n_fx, 1), np.int32)
        cf = np.zeros(max(n_cfg, 1), np.uint64)
        tot = np.zeros(4, np.uint64)
        L.refo_plan_export(self.handle, _p(steps, C.c_int64), _p(sl, C.c_int), _p(br, C.c_int),
                           _p(fx, C.c_int), _p(cf, C.c_uint64), _p(tot, C.c_uint64))
        self.plan = dict(steps=steps[:n_steps], sliced=sl[:n_sl], broken=br[:n_br],
                         fixed_outputs=fx[:n_fx], configs=cf[:n_cfg],
                         flops_per_slice=int(tot[0]), traffic_bytes_per_slice=int(tot[1]),
                         peak_bytes=int(tot[2]), memory_budget_bytes=int(tot[3]))

    # ---- hot-path calls
    @property
    def n_open(self):
        return len(self.net["open_labels"])

    def contract_group(self, fixed_bits: int) -> np.ndarray:
        out = np.zeros(2 << self.n_open, np.float64)
        _check(lib().refo_contract_group(self.handle, C.c_uint64(fixed_bits), _p(out, C.c_double)))
        return _cplx(out)

    def contract(self, fixed: dict | None = None, configs=None, workers: int = 1):
        fixed = fixed or {}
        fl = _ints(list(fixed.keys()) or [0])
        fv = _ints(list(fixed.values()) or [0])
        cf = _u64(configs if configs is not None else [0])
        n_cfg = 0 if configs is None else len(configs)
        n_free = len(self.net["open_labels"])
        out = np.zeros(2 << n_free, np.float64)
        flops = C.c_uint64()
        _check(lib().refo_contract(self.handle, len(fixed), _p(fl, C.c_int), _p(fv, C.c_int), n_cfg,
                                   _p(cf, C.c_uint64), workers, _p(out, C.c_double), C.byref(flops)))
        return _cplx(out), flops.value

    def execute_gsc(self, fixed_bits: int, slice_idx: int, config_bits: int = 0) -> np.ndarray:
        out = np.zeros(2 << self.n_open, np.float64)
        _check(lib().refo_execute_gsc(self.handle, C.c_uint64(fixed_bits), C.c_uint64(slice_idx),
                                      C.c_uint64(config_bits), _p(out, C.c_double)))
        return _cplx(out)

    def execute(self, assignment: dict) -> np.ndarray:
        ls = _ints(list(assignment.keys()) or [0])
        vs = _ints(list(assignment.values()) or [0])
        n = C.c_int64()
        _check(lib().refo_execute(self.handle, len(assignment), _p(ls, C.c_int), _p(vs, C.c_int),
                                  None, C.byref(n)))
        out = np.zeros(2 * n.value, np.float64)
        _check(lib().refo_execute(self.handle, len(assignment), _p(ls, C.c_int), _p(vs, C.c_int),
                                  _p(out, C.c_double), C.byref(n)))
        return _cplx(out)

    def plan_json(self) -> str:
        """plan_to_json (contraction_plan.cpp:451-491) of this problem's plan."""
        n = lib().refo_plan_json(self.handle, None, 0)
        buf = C.create_string_buffer(int(n) + 1)
        lib().refo_plan_json(self.handle, buf, n + 1)
        return buf.value.decode()

    def set_plan(self, steps, sliced):
        """Run an imported plan (steps [n][3], sliced labels) on the reference executor."""
        st = np.ascontiguousarray(np.asarray(steps, np.int64)[:, :3].reshape(-1), np.int32)
        sl = _ints(list(sliced) or [0])
        _check(lib().refo_set_plan(self.handle, len(st) // 3, _p(st, C.c_int), len(sliced), _p(sl, C.c_int)))
        self.plan["steps"] = np.asarray(steps)
        self.plan["sliced"] = np.asarray(sliced)

    def exact(self, cap: int = 24) -> np.ndarray:
        out = np.zeros(2 << self.n, np.float64)
        _check(lib().refo_exact(self.handle, cap, _p(out, C.c_double)))
        return _cplx(out)

    def gates(self) -> np.ndarray:
        n = lib().refo_circuit_gates(self.handle, None)
        out = np.zeros(4 * n, np.int32)
        lib().refo_circuit_gates(self.handle, _p(out, C.c_int))
        return out.reshape(-1, 4)

    def groups_mt(self, fixed: np.ndarray, threads: int):
        fixed = _u64(fixed)
        out = np.zeros(2 * (len(fixed) << self.n_open), np.float64)
        secs = C.c_double()
        _check(lib().refo_groups_mt(self.handle, _p(fixed, C.c_uint64), len(fixed), threads,
                                    _p(out, C.c_double), C.byref(secs)))
        return _cplx(out).reshape(len(fixed), -1), secs.value

    def slices_mt(self, fixed_bits: int, slices, threads: int):
        sl = _u64(slices)
        out = np.zeros(2 * (len(sl) << self.n_open), np.float64)
        secs = C.c_double()
        _check(lib().refo_slices_mt(self.handle, C.c_uint64(fixed_bits), _p(sl, C.c_uint64), len(sl),
                                    threads, _p(out, C.c_double), C.byref(secs)))
        return _cplx(out).reshape(len(sl), -1), secs.value


# ---- sampler
def candidates(n: int, open_qubits, n_groups: int, seed: int):
    op = _ints(sorted(open_qubits))
    out = np.zeros(n_groups, np.uint64)
    dup = C.c_int()
    _check(lib().refo_candidates(n, _p(op, C.c_int), len(op), C.c_uint64(n_groups), C.c_uint64(seed),
                                 _p(out, C.c_uint64), C.byref(dup)))
    return out, dup.value


def member(n: int, open_qubits, fixed: int, i: int) -> int:
    op = _ints(sorted(open_qubits))
    return int(lib().refo_member(n, _p(op, C.c_int), len(op), C.c_uint64(fixed), C.c_uint64(i)))


def top_k(n, open_qubits, fixed, probs, k):
    op = _ints(sorted(open_qubits))
    fixed = _u64(fixed)
    probs = np.ascontiguousarray(probs, np.float64)
    out = np.zeros(k, np.uint64)
    _check(lib().refo_topk(n, _p(op, C.c_int), len(op), len(fixed), _p(fixed, C.c_uint64),
                           _p(probs, C.c_double), C.c_uint64(k), _p(out, C.c_uint64)))
    return out


def direct(n, open_qubits, fixed, probs, seed):
    op = _ints(sorted(open_qubits))
    fixed = _u64(fixed)
    probs = np.ascontiguousarray(probs, np.float64)
    out = np.zeros(len(fixed), np.uint64)
    _check(lib().refo_direct(n, _p(op, C.c_int), len(op), len(fixed), _p(fixed, C.c_uint64),
                             _p(probs, C.c_double), C.c_uint64(seed), _p(out, C.c_uint64)))
    return out


def xeb(n, samples, q):
    s = _u64(samples)
    q = np.ascontiguousarray(q, np.float64)
    out = C.c_double()
    _check(lib().refo_xeb(n, _p(s, C.c_uint64), len(s), _p(q, C.c_double), C.byref(out)))
    return out.value


def split_next(seed: int, tag: int) -> int:
    return int(lib().refo_rng_split_next(C.c_uint64(seed), C.c_uint64(tag)))


def lexkey(index: int, n: int) -> int:
    return int(lib().refo_lexkey(C.c_uint64(index), n))


def timings_csv(ids, bits, ms, flops) -> str:
    ids, bits, flops = _u64(ids), _u64(bits), _u64(flops)
    ms = np.ascontiguousarray(ms, np.float64)
    n = lib().refo_timings_csv(len(ids), _p(ids, C.c_uint64), _p(bits, C.c_uint64), _p(ms, C.c_double),
                               _p(flops, C.c_uint64), None, 0)
    buf = C.create_string_buffer(int(n) + 1)
    lib().refo_timings_csv(len(ids), _p(ids, C.c_uint64), _p(bits, C.c_uint64), _p(ms, C.c_double),
                           _p(flops, C.c_uint64), buf, n + 1)
    return buf.value.decode()


def samples_text(n_qubits, topk, k, samples) -> str:
    s = _u64(samples)
    n = lib().refo_samples_text(n_qubits, int(topk), C.c_uint64(k), len(s), _p(s, C.c_uint64), None, 0)
    buf = C.create_string_buffer(int(n) + 1)
    lib().refo_samples_text(n_qubits, int(topk), C.c_uint64(k), len(s), _p(s, C.c_uint64), buf, n + 1)
    return buf.value.decode()
