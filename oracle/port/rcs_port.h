/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference hot path.
 *
 * This is the CHECKER the GPU parity tests compare against (and which
 * tests/test_oracle.py pins against the reference library itself,
 * oracle/_ref/librcs_ref.so, and against tests/golden/ fixtures).  It is never
 * linked into the product library (paper_2406_18889_b200/), and the product
 * never calls it.
 *
 * Every function cites the reference file:line it restates
 * (/root/reference/proj/...).
 */
#ifndef RCS_PORT_H
#define RCS_PORT_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Flat network + plan (the same data the reference's TensorNetwork and
 * ContractionPlan hold, include/rcs/tensor_network.hpp:14-43,
 * include/rcs/contraction_plan.hpp:11-36). Leaf data: row-major, labels[0] is
 * the most significant bit, interleaved (re, im) doubles, leaves concatenated. */
typedef struct port_net {
    int n_leaves;
    const int* leaf_rank;    /* [n_leaves] */
    const int* leaf_labels;  /* concatenated labels */
    const double* leaf_data; /* concatenated 2^rank complex per leaf */
    int n_labels;
    int n_qubits;
    const int* output_labels; /* [n_qubits] */
    int n_open;
    const int* open_labels; /* [n_open], ascending qubit order */
    const int* open_qubits; /* [n_open], ascending */
    int n_steps;
    const int* steps; /* [n_steps][3] lhs, rhs, result */
    int n_sliced;
    const int* sliced;
    int n_broken;
    const int* broken;
} port_net;

/* status codes = the reference's exit codes (include/rcs/errors.hpp:9-25) */
enum { PORT_OK = 0, PORT_CONFIG = 2, PORT_NUMERIC = 3, PORT_CAPACITY = 4 };

const char* port_last_error(int* step);

/* SplitMix64, include/rcs/rng.hpp:14-41 */
uint64_t port_rng_next(uint64_t* state);
uint64_t port_rng_split(uint64_t state, uint64_t tag);
uint64_t port_rng_below(uint64_t* state, uint64_t bound);
double port_rng_double(uint64_t* state);

/* execute_assignment, contraction_engine.cpp:153-208.
 * assign[label] = -1 (free) / 0 / 1. out: 2^(#free) interleaved complex. */
int port_execute(const port_net* net, const int* assign, double* out, int64_t* n_out,
                 uint64_t* flops);

/* contract / contract_group, contraction_engine.cpp:210-325: group pinned by
 * fixed_bits (bit b <-> b-th non-open qubit), slices [s0, s1) summed in
 * ascending order, configurations summed with the compensated reduction in
 * list order. n_cfg == 0 means no broken edges. */
int port_contract_group(const port_net* net, uint64_t fixed_bits, int n_cfg,
                        const uint64_t* cfgs, uint64_t s0, uint64_t s1, double* out);

/* make_broken_config, contraction_engine.cpp:136-151 */
int port_broken_configs(int k, uint64_t m, uint64_t seed, uint64_t* out);

/* build_candidate_set, sampling.cpp:29-60 (open must be ascending) */
int port_candidates(int n, const int* open, int l, uint64_t n_groups, uint64_t seed,
                    uint64_t* out_fixed, int* duplicates);
/* CandidateSet::member, sampling.cpp:14-27 */
uint64_t port_member(int n, const int* open, int l, uint64_t fixed, uint64_t i);
/* lexicographic_key, sampling.cpp:75-80 */
uint64_t port_lexkey(uint64_t index, int n);

/* top_k_select, sampling.cpp:82-114. probs: [n_groups][2^l]. */
int port_topk(int n, const int* open, int l, uint64_t n_groups, const uint64_t* fixed,
              const double* probs, uint64_t k, uint64_t* out);
/* direct_sample, sampling.cpp:116-145 */
int port_direct(int n, const int* open, int l, uint64_t n_groups, const uint64_t* fixed,
                const double* probs, uint64_t seed, uint64_t* out);
/* xeb, sampling.cpp:62-73; q[i] = ideal probability of samples[i] */
int port_xeb(int n, uint64_t count, const double* q, double* out);

/* simulate_exact, statevector.cpp:27-87 from a gate list
 * (kind 0..3 = SqrtX, SqrtY, SqrtW, fSim; q1 = -1 for 1-qubit gates). */
int port_statevector(int n, int n_gates, const int* kinds, const int* q0, const int* q1,
                     double* out);

#ifdef __cplusplus
}
#endif
#endif
