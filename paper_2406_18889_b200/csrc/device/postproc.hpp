// Post-processing entry points (see postproc.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "rcsg.h"

namespace rcsg {

struct PostResult {
    double device_ms = 0;           // CUDA-event time of the device work
    uint64_t bytes = 0;             // algorithmic bytes: candidates read once + samples written
    uint64_t candidates_kept = 0;   // entries the threshold pass kept (total on the full path)
    bool fast_path = false;         // threshold select (false: full sort)
    bool fallback = false;          // threshold missed, redone with the full sort
    double xeb_top = 0, xeb_direct = 0;  // when a device statevector was given
};

// Fused post-processing of DEVICE amplitudes (from_amps) or probabilities
// [G][2^l]: top-k (out_top != nullptr), direct sampling (want_direct) and, with
// a device statevector d_state (2^n interleaved complex f64), the XEB of both
// sample sets.  Outputs go to host memory, or device memory if device_out.
// force_path: 0 auto, 1 threshold select, 2 full sort (tests).
PostResult postprocess(const rcsg_candidates& cs, const double* d_src, bool from_amps, uint64_t k,
                       uint64_t* out_top, bool want_direct, uint64_t seed, uint64_t* out_direct,
                       const double* d_state, bool device_out, int force_path);

void topk_select(const rcsg_candidates& cs, const double* d_src, bool from_amps, uint64_t k,
                 uint64_t* out, cudaStream_t st);
void direct_sample(const rcsg_candidates& cs, const double* d_src, bool from_amps, uint64_t seed,
                   uint64_t* out, cudaStream_t st);
// (2^n / count) * sum q - 1 with q = |d_state[indices[i]]|^2 (HOST indices), or
// q = d_q[i] (device) when d_state is null; fixed-shape device reduction.
double xeb_device(int n_qubits, uint64_t count, const double* d_state, const uint64_t* indices,
                  const double* d_q);
}  // namespace rcsg
