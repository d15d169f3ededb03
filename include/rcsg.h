/* rcsg.h — C ABI of the B200-native contraction + sampling path.
 *
 * Plain C types only (pointers, sizes, status codes); no torch / C++ types.
 * This is the boundary the host C++ API (rcs_b200.hpp, namespace rcs) calls,
 * and what a reference-side FFI (ctypes / pybind / dlopen) binds; see
 * INTEGRATION.md.  Each entry point names the reference interface it replaces
 * (file:line into /root/reference/proj).
 *
 * Status codes mirror the reference's error taxonomy (include/rcs/errors.hpp:9-25):
 *   0 ok, 2 ConfigError, 3 NumericFault (step index via rcsg_last_error),
 *   4 CapacityError, 5 CUDA/NCCL runtime failure.
 *
 * Layout conventions (parity-critical):
 *   - leaf data row-major, labels[0] = most significant index bit, complex as
 *     interleaved (re, im) float64;
 *   - amplitudes of a group: bit j of the index <-> j-th smallest open qubit
 *     (contraction_engine.cpp:193-207);
 *   - group fixed bits: bit b <-> b-th non-open qubit in ascending order
 *     (contraction_engine.cpp:310-318, sampling.cpp:14-27);
 *   - slice s: bit b <-> plan.sliced[b]; broken config: bit b <-> plan.broken[b]
 *     (contraction_engine.cpp:242-248).
 */
#ifndef RCSG_H
#define RCSG_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    RCSG_OK = 0,
    RCSG_ERR_CONFIG = 2,
    RCSG_ERR_NUMERIC = 3,
    RCSG_ERR_CAPACITY = 4,
    RCSG_ERR_DEVICE = 5
};

/* Arithmetic of the contraction kernels. */
enum {
    RCSG_PREC_F64 = 0,   /* fp64 SIMT: reference-grade (<= 1e-10 norm-relative) */
    RCSG_PREC_F32 = 1,   /* fp32 SIMT */
    RCSG_PREC_TF32 = 2,  /* tcgen05 kind::tf32, fp32 accumulate in TMEM */
    RCSG_PREC_3XTF32 = 3, /* fp32 storage, split hi + lo operands on tcgen05 kind::tf32 (fp32-grade) */
    RCSG_PREC_BF16 = 4,   /* bf16 storage, tcgen05 kind::f16 (BF16 operands), fp32 accumulate */
    RCSG_PREC_F16 = 5     /* fp16 storage with calibrated per-tensor 2^e scales, kind::f16, fp32 accumulate */
};

/* TensorNetwork (tensor_network.hpp:26-43), flattened. */
typedef struct rcsg_network_desc {
    int32_t n_leaves;
    const int32_t* leaf_rank;   /* [n_leaves] */
    const int32_t* leaf_labels; /* concatenated, sum(rank) */
    const double* leaf_data;    /* concatenated 2^rank complex (interleaved) */
    int32_t n_labels;
    int32_t n_qubits;
    const int32_t* output_labels; /* [n_qubits] final wire label per qubit */
    int32_t n_open;
    const int32_t* open_labels; /* [n_open], ascending qubit */
    const int32_t* open_qubits; /* [n_open], ascending */
} rcsg_network_desc;

/* ContractionPlan (contraction_plan.hpp:19-36), flattened. */
typedef struct rcsg_plan_desc {
    int32_t n_steps;
    const int32_t* steps; /* [n_steps][3] = lhs, rhs, result node ids (post-order) */
    int32_t n_sliced;
    const int32_t* sliced;
    int32_t n_broken;
    const int32_t* broken;
    int32_t n_fixed;
    const int32_t* fixed_outputs;
} rcsg_plan_desc;

typedef struct rcsg_stats {
    uint64_t plan_flops;       /* sum over assignments of plan.flops_per_slice (reference-equivalent) */
    uint64_t executed_flops;   /* 8*m*k*n actually issued on the device (after group sharing) */
    uint64_t arena_bytes;      /* device arena size */
    uint64_t kernel_launches;  /* our kernels launched */
    uint64_t passes;           /* (config, slice, group-chunk) passes */
    double device_ms;          /* CUDA-event time of the contraction on the program's stream */
    /* filled only when profiling is on (rcsg_program_set_profile): CUDA-event
     * time of each kernel class on the program's stream, plus its work */
    double gemm_ms;            /* complex GEMM launches (tensor-core + SIMT) */
    double gemm_tc_ms;         /* tensor-core (tcgen05) GEMM launches only */
    uint64_t gemm_tc_flops;    /* 8*m*n*k issued by tensor-core launches */
    double permute_ms;         /* bit-permutation launches */
    uint64_t permute_bytes;    /* bytes read + written by permutes */
    uint64_t gemm_tc_launches;
    /* the single longest launch of the profiled run (roofline of the dominant
     * kernel): its time, algorithmic FLOPs and bytes (operands read once +
     * result written once, at storage precision), plan step and kernel class
     * (0 SIMT GEMM, 1 tensor-core GEMM, 2 permute, 3 GEMV) */
    double top_ms;
    uint64_t top_flops;
    uint64_t top_bytes;
    int64_t top_step;
    int64_t top_class;
    double top_ms_sum;     /* summed time and count of every launch of plan step top_step */
                           /* (same kernel class) in the profiled run: the average launch */
    uint64_t top_launches;
} rcsg_stats;

typedef struct rcsg_program rcsg_program;

/* Last error message of this thread; *step = NumericFault step index or -1. */
const char* rcsg_last_error(int32_t* step);

/* Bind the calling thread to CUDA device `device` (one process per GPU). */
int rcsg_set_device(int32_t device);

/* Compile (network, plan) into a device step program.  Deep-copies the
 * descriptors (the plan stays immutable, contraction_plan.hpp:17-18).
 * `mem_budget_bytes` bounds the device arena (0 = 70% of free memory).
 * Replaces: the per-call interpretation of the plan in contract()
 * (contraction_engine.cpp:153-208). */
int rcsg_compile(const rcsg_network_desc* net, const rcsg_plan_desc* plan, int32_t precision,
                 uint64_t mem_budget_bytes, rcsg_program** out);
int rcsg_program_free(rcsg_program* prog);

/* Per-kernel-class CUDA-event timing (fills the *_ms fields of rcsg_stats).
 * Adds two event records per launch; off by default. */
int rcsg_program_set_profile(rcsg_program* prog, int32_t on);

/* The CUDA stream (cudaStream_t) the program launches on, for callers that
 * time it with their own events or order work after it. */
int rcsg_program_stream(rcsg_program* prog, void** out);

/* Amplitudes of n_groups candidate groups: for each group g,
 *   sum over configs (compensated, list order) of
 *   sum over slices s in [slice_begin, slice_end) (ascending)
 * of the plan executed under (group_fixed[g], slice s, config).
 * n_configs == 0: exact contraction (the plan must have no broken edges).
 * out_amps: HOST [n_groups][2^l] interleaved float64.
 * Replaces: contract_group (contraction_engine.cpp:307-325) and contract()
 * with fixed_outputs (:210-305), batched over groups. */
int rcsg_contract_groups(rcsg_program* prog, uint64_t n_groups, const uint64_t* group_fixed,
                         uint64_t n_configs, const uint64_t* configs, uint64_t slice_begin,
                         uint64_t slice_end, double* out_amps, rcsg_stats* stats);

/* Same, but accumulates (+=) into a DEVICE buffer d_acc [n_groups][2^l]
 * interleaved float64 on the program's stream, without host synchronisation
 * when `sync` == 0.  Used by the slice scheduler (one call per rank shard)
 * before the cross-GPU reduction. */
int rcsg_contract_groups_device(rcsg_program* prog, uint64_t n_groups,
                                const uint64_t* group_fixed, uint64_t n_configs,
                                const uint64_t* configs, uint64_t slice_begin,
                                uint64_t slice_end, double* d_acc, int32_t sync,
                                rcsg_stats* stats);

/* Wait for the program's stream; reports (RCSG_ERR_NUMERIC) a non-finite
 * intermediate of an earlier sync == 0 call. */
int rcsg_program_sync(rcsg_program* prog);

/* Compile with explicit pins instead of group variants: pinned[label] in {0,1}
 * fixes a label for every execution (-1 = not pinned); sliced / broken labels
 * still come from the pass.  Every non-open output must be pinned, otherwise
 * RCSG_ERR_CONFIG ("assignment incomplete").  Run it with one group (fixed
 * bits ignored).  Serves contract() with arbitrary fixed_outputs
 * (contraction_engine.cpp:210-305). */
int rcsg_compile_pinned(const rcsg_network_desc* net, const rcsg_plan_desc* plan, int32_t precision,
                        uint64_t mem_budget_bytes, const int8_t* pinned, rcsg_program** out);

/* execute_assignment (contraction_engine.cpp:153-208): every label with
 * assign[label] in {0,1} pinned, -1 free.  out: host, 2^(#free) complex in
 * canonical open-qubit order; *n_out = count.  Free labels must be open outputs. */
int rcsg_execute_assignment(const rcsg_network_desc* net, const rcsg_plan_desc* plan,
                            int32_t precision, const int8_t* assign, double* out,
                            uint64_t* n_out);

/* ---- multi-GPU context (one host thread, all local GPUs, NCCL) -------------- */

/* One process drives the listed local GPUs: a stream per device and one NCCL
 * communicator clique over them (ncclCommInitAll over NVLink / NVSwitch; NCCL
 * is loaded at run time).  Replaces the reference's worker thread pool of
 * contract() (contraction_engine.cpp:264-287) with devices. */
typedef struct rcsg_context rcsg_context;
typedef struct rcsg_multi rcsg_multi;
int rcsg_init(const int32_t* devices, int32_t n_devices, rcsg_context** out);
int rcsg_context_free(rcsg_context* ctx);
int rcsg_context_devices(rcsg_context* ctx, int32_t* n_devices);

/* Compile (network, plan) on every device of the context.  n_blocks: canonical
 * slice blocks (0 = 8). */
int rcsg_context_compile(rcsg_context* ctx, const rcsg_network_desc* net, const rcsg_plan_desc* plan,
                         int32_t precision, uint64_t mem_budget_bytes, int32_t n_blocks, rcsg_multi** out);
int rcsg_multi_free(rcsg_multi* m);

/* rcsg_contract_groups over the first n_used devices (0 = all): the slice range
 * is cut into the program's canonical blocks (independent of n_used), blocks go
 * to devices round-robin, each device sums its blocks' slices in ascending
 * order into device partials, the partials are gathered to the first device
 * with NCCL and added in block order - bit-identical for any n_used (the
 * reference's worker-count invariance, test_contraction.cpp:84-93).
 * out_amps: HOST [n_groups][2^l] interleaved float64. */
int rcsg_multi_contract_groups(rcsg_multi* m, uint64_t n_groups, const uint64_t* group_fixed, uint64_t n_configs,
                               const uint64_t* configs, uint64_t slice_begin, uint64_t slice_end, int32_t n_used,
                               double* out_amps, rcsg_stats* stats);

/* ---- exact statevector (XEB oracle) ----------------------------------------- */

/* simulate_exact (statevector.cpp:79-86) on the device: |0..0> followed by the
 * gates in order.  Gate g acts on n_targets[g] (1 or 2) qubits targets[2g],
 * targets[2g+1] with the row-major unitary at unitaries[32g ..] (16 interleaved
 * complex f64; a 1-qubit gate uses the first 4).  Basis of a 2-qubit block:
 * (bit of targets[2g]) << 1 | bit of targets[2g+1] (statevector.cpp:42).
 * d_state: DEVICE buffer of 2^n interleaved complex f64 (qubit q = index bit
 * q).  Products and sums are rounded in the reference's order.
 * Replaces: simulate_exact / apply_gate (statevector.hpp:29, statevector.cpp:60-86). */
int rcsg_statevector(int32_t n_qubits, int32_t n_gates, const int32_t* n_targets, const int32_t* targets,
                     const double* unitaries, double* d_state);

/* |amplitude|^2 at the given basis indices of a device statevector (HOST
 * indices in, HOST probabilities out).  Replaces: ideal_probability
 * (statevector.hpp:32). */
int rcsg_statevector_probs(const double* d_state, uint64_t n_indices, const uint64_t* indices, double* out);

/* ---- post-processing (sampling.cpp) on device amplitudes ------------------ */

/* Candidate-set description (CandidateSet, sampling.hpp:17-31). */
typedef struct rcsg_candidates {
    int32_t n_qubits;
    int32_t l;
    const int32_t* open_qubits; /* [l] ascending */
    uint64_t n_groups;
    const uint64_t* group_fixed; /* HOST [n_groups] */
} rcsg_candidates;

/* top_k_select (sampling.cpp:82-114): global top-k of |a|^2 over all
 * n_groups*2^l candidates, ordered by (prob desc, lexicographic asc).
 * d_amps: DEVICE [n_groups][2^l] interleaved float64.  out: HOST k indices. */
int rcsg_topk(const rcsg_candidates* cs, const double* d_amps, uint64_t k, uint64_t* out);

/* Same selection from DEVICE probabilities [n_groups][2^l] (the reference's
 * ProbFn values), bit-exact with top_k_select on identical inputs. */
int rcsg_topk_probs(const rcsg_candidates* cs, const double* d_probs, uint64_t k, uint64_t* out);

/* direct_sample (sampling.cpp:116-145): one inverse-CDF draw per group with the
 * counter-based SplitMix64 stream of rng_seed.  out: HOST [n_groups]. */
int rcsg_direct_sample(const rcsg_candidates* cs, const double* d_amps, uint64_t rng_seed,
                       uint64_t* out);

int rcsg_direct_sample_probs(const rcsg_candidates* cs, const double* d_probs, uint64_t rng_seed,
                             uint64_t* out);

/* xeb (sampling.cpp:62-73): (2^n / count) * sum q - 1 over HOST q[count]
 * (reduced on the device in a fixed order; equals the reference's sequential
 * sum to ~1e-15 relative).  q must be finite and >= 0, else RCSG_ERR_CONFIG. */
int rcsg_xeb(int32_t n_qubits, uint64_t count, const double* q, double* out);

/* xeb with the ideal probabilities read on the device: q = |d_state[idx]|^2 of
 * a DEVICE statevector (2^n interleaved complex f64, e.g. from
 * rcsg_statevector) at the HOST sample indices.  Replaces xeb(samples,
 * ideal_probability) (sampling.cpp:62-73, statevector.hpp:32). */
int rcsg_xeb_state(int32_t n_qubits, uint64_t count, const uint64_t* indices, const double* d_state,
                   double* out);

/* Result of rcsg_postprocess. */
typedef struct rcsg_post_stats {
    double device_ms;          /* CUDA-event time of the device work */
    uint64_t bytes;            /* algorithmic bytes: amplitudes read once + samples written */
    uint64_t candidates_kept;  /* candidates the threshold pass kept (all on the full-sort path) */
    int32_t fast_path;         /* 1: threshold select; 0: full sort of every candidate */
    int32_t fallback;          /* 1: the threshold missed and the full sort ran instead */
    double xeb_topk;           /* with d_state: XEB of the top-k samples */
    double xeb_direct;         /* with d_state: XEB of the direct samples */
} rcsg_post_stats;

/* Fused post-processing of DEVICE amplitudes [n_groups][2^l] (interleaved f64):
 * |a|^2, global top-k (out_topk: HOST k indices, or NULL to skip) ordered as
 * top_k_select (sampling.cpp:82-114), one direct sample per group when
 * `direct` != 0 (out_direct: HOST [n_groups], sampling.cpp:116-145) — both from
 * one streaming pass over the amplitudes — and, when d_state (a DEVICE
 * statevector of the circuit) is given, the linear XEB of both sample sets
 * reduced on the device (sampling.cpp:62-73). */
int rcsg_postprocess(const rcsg_candidates* cs, const double* d_amps, uint64_t k, uint64_t* out_topk,
                     int32_t direct, uint64_t rng_seed, uint64_t* out_direct, const double* d_state,
                     rcsg_post_stats* stats);

/* Device buffers for the post-processing entry points (thin cudaMalloc wrappers
 * so FFI callers need no CUDA runtime of their own). */
int rcsg_device_alloc(uint64_t bytes, void** out);
int rcsg_device_free(void* p);
int rcsg_memcpy(void* dst, const void* src, uint64_t bytes, int32_t kind /*1 H2D, 2 D2H, 3 D2D*/);

#ifdef __cplusplus
}
#endif
#endif
