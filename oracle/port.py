"""TEST INFRASTRUCTURE ONLY — ctypes driver for the plain-C restatement
(oracle/port/rcs_port.c, built into oracle/_ref/librcs_port.so by oracle/Makefile).

Takes the same flat network/plan dicts that ``oracle.ref.RefProblem`` and
``paper_2406_18889_b200.Problem`` export, so the checker runs exactly the plan
the GPU ran.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "librcs_port.so")
_lib = None


class PortError(RuntimeError):
    def __init__(self, code, msg, step):
        super().__init__(f"[{code}] {msg}")
        self.code, self.msg, self.step = code, msg, step


class port_net(C.Structure):
    _fields_ = [("n_leaves", C.c_int), ("leaf_rank", C.POINTER(C.c_int)),
                ("leaf_labels", C.POINTER(C.c_int)), ("leaf_data", C.POINTER(C.c_double)),
                ("n_labels", C.c_int), ("n_qubits", C.c_int), ("output_labels", C.POINTER(C.c_int)),
                ("n_open", C.c_int), ("open_labels", C.POINTER(C.c_int)),
                ("open_qubits", C.POINTER(C.c_int)), ("n_steps", C.c_int),
                ("steps", C.POINTER(C.c_int)), ("n_sliced", C.c_int), ("sliced", C.POINTER(C.c_int)),
                ("n_broken", C.c_int), ("broken", C.POINTER(C.c_int))]


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle port`")
        L = C.CDLL(LIB_PATH)
        L.port_last_error.restype = C.c_char_p
        for n in ("port_rng_next", "port_rng_split", "port_rng_below", "port_member", "port_lexkey"):
            getattr(L, n).restype = C.c_uint64
        L.port_rng_double.restype = C.c_double
        _lib = L
    return _lib


def _check(rc):
    if rc:
        step = C.c_int(-1)
        msg = lib().port_last_error(C.byref(step)).decode()
        raise PortError(rc, msg, step.value)


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


class PortNet:
    """Holds the arrays behind a port_net built from exported net/plan dicts."""

    def __init__(self, net: dict, plan: dict):
        i32 = lambda x: np.ascontiguousarray(np.asarray(x, np.int32).reshape(-1) if len(x) else np.zeros(1, np.int32))
        self.rank = i32(net["leaf_rank"])
        self.labels = i32(net["leaf_labels"])
        self.data = np.ascontiguousarray(np.asarray(net["leaf_data"], np.float64))
        self.out_l = i32(net["output_labels"])
        self.open_l = i32(net["open_labels"])
        self.open_q = i32(net["open_qubits"])
        st = np.asarray(plan["steps"], np.int64)
        self.steps = i32(st[:, :3].reshape(-1)) if len(st) else np.zeros(1, np.int32)
        self.sliced = i32(plan["sliced"])
        self.broken = i32(plan["broken"])
        self.n_open = len(net["open_labels"])
        self.n_labels = int(net["n_labels"])
        self.net = port_net(len(net["leaf_rank"]), _p(self.rank, C.c_int), _p(self.labels, C.c_int),
                            _p(self.data, C.c_double), self.n_labels, int(net["n_qubits"]),
                            _p(self.out_l, C.c_int), self.n_open, _p(self.open_l, C.c_int),
                            _p(self.open_q, C.c_int), len(st), _p(self.steps, C.c_int),
                            len(plan["sliced"]), _p(self.sliced, C.c_int), len(plan["broken"]),
                            _p(self.broken, C.c_int))

    def contract_group(self, fixed_bits: int, configs=None, slices=None) -> np.ndarray:
        cf = np.ascontiguousarray(np.asarray(configs if configs is not None else [0], np.uint64))
        n_cfg = 0 if configs is None else len(cf)
        s0, s1 = slices if slices is not None else (0, 1 << self.net.n_sliced)
        out = np.zeros(2 << self.n_open, np.float64)
        _check(lib().port_contract_group(C.byref(self.net), C.c_uint64(fixed_bits), n_cfg,
                                         _p(cf, C.c_uint64), C.c_uint64(s0), C.c_uint64(s1),
                                         _p(out, C.c_double)))
        return out.view(np.complex128)

    def execute(self, assignment: dict) -> np.ndarray:
        a = np.full(self.n_labels, -1, np.int32)
        for k, v in assignment.items():
            a[int(k)] = int(v)
        n = C.c_int64()
        flops = C.c_uint64()
        out = np.zeros(2 << self.n_open, np.float64)
        _check(lib().port_execute(C.byref(self.net), _p(a, C.c_int), _p(out, C.c_double), C.byref(n),
                                  C.byref(flops)))
        return out[:2 * n.value].view(np.complex128)


def candidates(n, open_qubits, n_groups, seed):
    op = np.ascontiguousarray(sorted(open_qubits), np.int32)
    out = np.zeros(n_groups, np.uint64)
    dup = C.c_int()
    _check(lib().port_candidates(n, _p(op, C.c_int), len(op), C.c_uint64(n_groups), C.c_uint64(seed),
                                 _p(out, C.c_uint64), C.byref(dup)))
    return out, dup.value


def top_k(n, open_qubits, fixed, probs, k):
    op = np.ascontiguousarray(sorted(open_qubits), np.int32)
    fixed = np.ascontiguousarray(fixed, np.uint64)
    probs = np.ascontiguousarray(probs, np.float64)
    out = np.zeros(k, np.uint64)
    _check(lib().port_topk(n, _p(op, C.c_int), len(op), C.c_uint64(len(fixed)), _p(fixed, C.c_uint64),
                           _p(probs, C.c_double), C.c_uint64(k), _p(out, C.c_uint64)))
    return out


def direct(n, open_qubits, fixed, probs, seed):
    op = np.ascontiguousarray(sorted(open_qubits), np.int32)
    fixed = np.ascontiguousarray(fixed, np.uint64)
    probs = np.ascontiguousarray(probs, np.float64)
    out = np.zeros(len(fixed), np.uint64)
    _check(lib().port_direct(n, _p(op, C.c_int), len(op), C.c_uint64(len(fixed)), _p(fixed, C.c_uint64),
                             _p(probs, C.c_double), C.c_uint64(seed), _p(out, C.c_uint64)))
    return out


def xeb(n, q):
    q = np.ascontiguousarray(q, np.float64)
    out = C.c_double()
    _check(lib().port_xeb(n, C.c_uint64(len(q)), _p(q, C.c_double), C.byref(out)))
    return out.value


def statevector(n, gates) -> np.ndarray:
    """gates: rows (layer, kind, q0, q1) as exported by Problem.gates()."""
    g = np.asarray(gates, np.int32)
    kinds = np.ascontiguousarray(g[:, 1])
    q0 = np.ascontiguousarray(g[:, 2])
    q1 = np.ascontiguousarray(g[:, 3])
    out = np.zeros(2 << n, np.float64)
    _check(lib().port_statevector(n, len(g), _p(kinds, C.c_int), _p(q0, C.c_int), _p(q1, C.c_int),
                                  _p(out, C.c_double)))
    return out.view(np.complex128)


def split_next(seed: int, tag: int) -> int:
    st = C.c_uint64(int(lib().port_rng_split(C.c_uint64(seed), C.c_uint64(tag))))
    return int(lib().port_rng_next(C.byref(st)))


def member(n, open_qubits, fixed, i):
    op = np.ascontiguousarray(sorted(open_qubits), np.int32)
    return int(lib().port_member(n, _p(op, C.c_int), len(op), C.c_uint64(fixed), C.c_uint64(i)))


def lexkey(index, n):
    return int(lib().port_lexkey(C.c_uint64(index), n))


def broken_configs(k, m, seed):
    out = np.zeros(m, np.uint64)
    _check(lib().port_broken_configs(k, C.c_uint64(m), C.c_uint64(seed), _p(out, C.c_uint64)))
    return out
