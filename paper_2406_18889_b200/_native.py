"""ctypes binding of the product library (C ABI: include/rcsg.h + host rcsh_*).

There is no fallback: if the in-tree library is missing the import fails
loudly.  Build it with ``__graft_entry__.build()`` (or ``make -C
paper_2406_18889_b200/csrc``).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_native", "libpaper_2406_18889_b200.so")

RCSG_OK, RCSG_ERR_CONFIG, RCSG_ERR_NUMERIC, RCSG_ERR_CAPACITY, RCSG_ERR_DEVICE = 0, 2, 3, 4, 5
PRECISIONS = {"f64": 0, "f32": 1, "tf32": 2, "3xtf32": 3, "bf16": 4, "f16": 5}


class rcsg_network_desc(C.Structure):
    _fields_ = [("n_leaves", C.c_int32), ("leaf_rank", C.POINTER(C.c_int32)),
                ("leaf_labels", C.POINTER(C.c_int32)), ("leaf_data", C.POINTER(C.c_double)),
                ("n_labels", C.c_int32), ("n_qubits", C.c_int32),
                ("output_labels", C.POINTER(C.c_int32)), ("n_open", C.c_int32),
                ("open_labels", C.POINTER(C.c_int32)), ("open_qubits", C.POINTER(C.c_int32))]


class rcsg_plan_desc(C.Structure):
    _fields_ = [("n_steps", C.c_int32), ("steps", C.POINTER(C.c_int32)),
                ("n_sliced", C.c_int32), ("sliced", C.POINTER(C.c_int32)),
                ("n_broken", C.c_int32), ("broken", C.POINTER(C.c_int32)),
                ("n_fixed", C.c_int32), ("fixed_outputs", C.POINTER(C.c_int32))]


class rcsg_stats(C.Structure):
    _fields_ = [("plan_flops", C.c_uint64), ("executed_flops", C.c_uint64),
                ("arena_bytes", C.c_uint64), ("kernel_launches", C.c_uint64),
                ("passes", C.c_uint64), ("device_ms", C.c_double), ("gemm_ms", C.c_double),
                ("gemm_tc_ms", C.c_double), ("gemm_tc_flops", C.c_uint64),
                ("permute_ms", C.c_double), ("permute_bytes", C.c_uint64),
                ("gemm_tc_launches", C.c_uint64), ("top_ms", C.c_double), ("top_flops", C.c_uint64),
                ("top_bytes", C.c_uint64), ("top_step", C.c_int64), ("top_class", C.c_int64),
                ("top_ms_sum", C.c_double), ("top_launches", C.c_uint64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class rcsg_candidates(C.Structure):
    _fields_ = [("n_qubits", C.c_int32), ("l", C.c_int32), ("open_qubits", C.POINTER(C.c_int32)),
                ("n_groups", C.c_uint64), ("group_fixed", C.POINTER(C.c_uint64))]


class rcsg_post_stats(C.Structure):
    _fields_ = [("device_ms", C.c_double), ("bytes", C.c_uint64), ("candidates_kept", C.c_uint64),
                ("fast_path", C.c_int32), ("fallback", C.c_int32), ("xeb_topk", C.c_double),
                ("xeb_direct", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


# exported symbols and their restypes (everything else returns int status)
RCSG_SYMBOLS = [
    "rcsg_last_error", "rcsg_set_device", "rcsg_compile", "rcsg_compile_pinned", "rcsg_program_free",
    "rcsg_program_set_profile", "rcsg_program_stream",
    "rcsg_contract_groups", "rcsg_contract_groups_device", "rcsg_execute_assignment", "rcsg_topk",
    "rcsg_topk_probs", "rcsg_direct_sample", "rcsg_direct_sample_probs", "rcsg_xeb",
    "rcsg_device_alloc", "rcsg_device_free", "rcsg_memcpy", "rcsg_program_sync", "rcsg_statevector",
    "rcsg_statevector_probs", "rcsg_xeb_state", "rcsg_postprocess", "rcsg_init", "rcsg_context_free",
    "rcsg_context_devices", "rcsg_context_compile", "rcsg_multi_free", "rcsg_multi_contract_groups",
]
RCSH_SYMBOLS = [
    "rcsh_last_error", "rcsh_build", "rcsh_build_network", "rcsh_free", "rcsh_net_sizes",
    "rcsh_net_export", "rcsh_label_names", "rcsh_wire_edges", "rcsh_plan_sizes", "rcsh_plan_export",
    "rcsh_circuit_gates", "rcsh_contract_groups", "rcsh_contract_groups_device", "rcsh_contract",
    "rcsh_execute", "rcsh_candidates", "rcsh_topk", "rcsh_direct", "rcsh_member",
    "rcsh_rng_split_next", "rcsh_lexkey", "rcsh_broken_configs", "rcsh_set_profile",
    "rcsh_program_stream", "rcsh_program_sync", "rcsh_statevector", "rcsh_build_ex", "rcsh_plan_import",
    "rcsh_state_fidelity", "rcsh_predicted_topk_xeb", "rcsh_release_programs",
]

_lib = None
_testkit = None
TESTKIT_PATH = os.path.join(HERE, "_native", "libpaper_2406_18889_b200_testkit.so")


def testkit():
    """GEMM self-test / benchmark helpers (csrc/device/gemm_bench.cu), a separate
    library next to the product one - tests and tools only."""
    global _testkit
    if _testkit is None:
        lib()
        _testkit = C.CDLL(TESTKIT_PATH)
        for name in ("rcsg_gemm_selftest", "rcsg_gemm_check_f16", "rcsg_gemm_check_bf16", "rcsg_gemm_check_tf32",
                     "rcsg_gemm_check_3xtf32",
                     "rcsg_gemm_bench_f16", "rcsg_gemm_bench_tf32"):
            getattr(_testkit, name).restype = C.c_int
    return _testkit


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"native library {LIB_PATH} is missing; build it with __graft_entry__.build() "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name in RCSG_SYMBOLS + RCSH_SYMBOLS:
            getattr(L, name).restype = C.c_int
        L.rcsg_last_error.restype = C.c_char_p
        L.rcsh_last_error.restype = C.c_char_p
        L.rcsh_free.restype = None
        L.rcsh_set_profile.restype = None
        L.rcsh_release_programs.restype = None
        L.rcsh_net_sizes.restype = None
        L.rcsh_net_export.restype = None
        L.rcsh_wire_edges.restype = None
        L.rcsh_plan_sizes.restype = None
        L.rcsh_plan_export.restype = None
        L.rcsh_label_names.restype = C.c_int64
        for name in ("rcsh_plan_json", "rcsh_timings_csv", "rcsh_samples_text", "rcsh_samples_parse"):
            getattr(L, name).restype = C.c_int64
        L.rcsh_circuit_gates.restype = C.c_int64
        L.rcsh_member.restype = C.c_uint64
        L.rcsh_rng_split_next.restype = C.c_uint64
        L.rcsh_lexkey.restype = C.c_uint64
        _lib = L
    return _lib
