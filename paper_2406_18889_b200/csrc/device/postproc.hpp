// Post-processing entry points (see postproc.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "rcsg.h"

namespace rcsg {
// d_src: device amplitudes [G][2^l] interleaved (from_amps) or probabilities [G][2^l].
void topk_select(const rcsg_candidates& cs, const double* d_src, bool from_amps, uint64_t k,
                 uint64_t* out, cudaStream_t st);
void direct_sample(const rcsg_candidates& cs, const double* d_src, bool from_amps, uint64_t seed,
                   uint64_t* out, cudaStream_t st);
}  // namespace rcsg
