// Exact statevector on the GPU: the reference's
// simulate_exact / apply_gate (statevector.cpp:20-86) for XEB oracles at
// n <= 33 (2^33 complex f64 = 137 GB of HBM).  One launch per gate; each
// thread updates one 2- or 4-amplitude group in place.  Products and sums are
// rounded separately in the reference's order (no FMA contraction), so the
// amplitudes match the reference's complex<double> arithmetic.
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "rcsg.h"

namespace rcsg {
namespace {

struct C2 {
    double re, im;
};
__device__ __forceinline__ C2 cmul(C2 a, C2 b) {  // (ac - bd) + (ad + bc) i, separately rounded
    return {__dsub_rn(__dmul_rn(a.re, b.re), __dmul_rn(a.im, b.im)),
            __dadd_rn(__dmul_rn(a.re, b.im), __dmul_rn(a.im, b.re))};
}
__device__ __forceinline__ C2 cadd(C2 a, C2 b) { return {__dadd_rn(a.re, b.re), __dadd_rn(a.im, b.im)}; }

// insert a zero bit at position b of x
__device__ __forceinline__ uint64_t ins0(uint64_t x, int b) {
    const uint64_t lo = x & ((uint64_t{1} << b) - 1);
    return ((x >> b) << (b + 1)) | lo;
}

__global__ void init_kernel(C2* s, uint64_t dim) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < dim;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        s[i] = {i == 0 ? 1.0 : 0.0, 0.0};
}

__global__ void gate1_kernel(C2* s, uint64_t groups, int q, C2 u0, C2 u1, C2 u2, C2 u3) {
    for (uint64_t g = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; g < groups;
         g += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t i = ins0(g, q), j = i | (uint64_t{1} << q);
        const C2 a0 = s[i], a1 = s[j];
        s[i] = cadd(cmul(u0, a0), cmul(u1, a1));
        s[j] = cadd(cmul(u2, a0), cmul(u3, a1));
    }
}

struct U4 {
    C2 u[16];
};
// basis within the block: (bit of qa) << 1 | bit of qb  (statevector.cpp:42)
__global__ void gate2_kernel(C2* s, uint64_t groups, int qa, int qb, const U4 u) {
    const int lo = qa < qb ? qa : qb, hi = qa < qb ? qb : qa;
    const uint64_t ba = uint64_t{1} << qa, bb = uint64_t{1} << qb;
    for (uint64_t g = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; g < groups;
         g += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t i = ins0(ins0(g, lo), hi);
        const uint64_t idx[4] = {i, i | bb, i | ba, i | ba | bb};
        C2 in[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) in[r] = s[idx[r]];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            C2 acc = cmul(u.u[4 * r], in[0]);
            acc = cadd(acc, cmul(u.u[4 * r + 1], in[1]));
            acc = cadd(acc, cmul(u.u[4 * r + 2], in[2]));
            acc = cadd(acc, cmul(u.u[4 * r + 3], in[3]));
            s[idx[r]] = acc;
        }
    }
}

__global__ void probs_kernel(const C2* s, const uint64_t* idx, int64_t n, double* out) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const C2 a = s[idx[t]];
        out[t] = __dadd_rn(__dmul_rn(a.re, a.re), __dmul_rn(a.im, a.im));
    }
}

int grid_for(uint64_t work) { return static_cast<int>(std::min<uint64_t>((work + 255) / 256, 148ull * 32)); }

}  // namespace
}  // namespace rcsg

using namespace rcsg;

extern "C" int rcsg_statevector(int32_t n_qubits, int32_t n_gates, const int32_t* n_targets, const int32_t* targets,
                                const double* unitaries, double* d_state) {
    try {
        if (n_qubits < 1 || n_qubits > 36) return RCSG_ERR_CAPACITY;
        if (!d_state || (n_gates && (!n_targets || !targets || !unitaries))) return RCSG_ERR_CONFIG;
        C2* s = reinterpret_cast<C2*>(d_state);
        const uint64_t dim = uint64_t{1} << n_qubits;
        init_kernel<<<grid_for(dim), 256>>>(s, dim);
        for (int gi = 0; gi < n_gates; ++gi) {
            const int nt = n_targets[gi];
            const int qa = targets[2 * gi], qb = targets[2 * gi + 1];
            const double* u = unitaries + 32 * static_cast<int64_t>(gi);  // 16 complex per gate (1q: first 4)
            if (qa < 0 || qa >= n_qubits || (nt == 2 && (qb < 0 || qb >= n_qubits || qb == qa)) || (nt != 1 && nt != 2))
                return RCSG_ERR_CONFIG;
            if (nt == 1) {
                gate1_kernel<<<grid_for(dim / 2), 256>>>(s, dim / 2, qa, C2{u[0], u[1]}, C2{u[2], u[3]},
                                                         C2{u[4], u[5]}, C2{u[6], u[7]});
            } else {
                U4 m;
                for (int r = 0; r < 16; ++r) m.u[r] = C2{u[2 * r], u[2 * r + 1]};
                gate2_kernel<<<grid_for(dim / 4), 256>>>(s, dim / 4, qa, qb, m);
            }
        }
        return cudaDeviceSynchronize() == cudaSuccess && cudaGetLastError() == cudaSuccess ? RCSG_OK
                                                                                           : RCSG_ERR_DEVICE;
    } catch (...) {
        return RCSG_ERR_DEVICE;
    }
}

extern "C" int rcsg_statevector_probs(const double* d_state, uint64_t n_indices, const uint64_t* indices,
                                      double* out) {
    try {
        if (!d_state || (n_indices && (!indices || !out))) return RCSG_ERR_CONFIG;
        if (n_indices == 0) return RCSG_OK;
        uint64_t* di;
        double* dout;
        if (cudaMalloc(&di, n_indices * 8) || cudaMalloc(&dout, n_indices * 8)) return RCSG_ERR_DEVICE;
        cudaMemcpy(di, indices, n_indices * 8, cudaMemcpyHostToDevice);
        probs_kernel<<<grid_for(n_indices), 256>>>(reinterpret_cast<const C2*>(d_state), di,
                                                   static_cast<int64_t>(n_indices), dout);
        cudaMemcpy(out, dout, n_indices * 8, cudaMemcpyDeviceToHost);
        cudaFree(di);
        cudaFree(dout);
        return cudaGetLastError() == cudaSuccess ? RCSG_OK : RCSG_ERR_DEVICE;
    } catch (...) {
        return RCSG_ERR_DEVICE;
    }
}
