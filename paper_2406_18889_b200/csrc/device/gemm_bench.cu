// Isolated complex-GEMM check + timing (C ABI rcsg_gemm_selftest), used by the
// GPU tests and the kernel-tuning scripts: random planar operands, tensor-core
// result vs the fp32 SIMT kernel, CUDA-event time per launch.
#include <cmath>
#include <cstdint>
#include <vector>

#include "executor.hpp"
#include "kernels.cuh"

namespace rcsg {
namespace {

__global__ void fill_rand(float* p, int64_t n, uint64_t seed) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        uint64_t z = seed + (i + 1) * 0x9e3779b97f4a7c15ull;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        z ^= z >> 31;
        p[i] = static_cast<float>(static_cast<double>(z >> 11) * 0x1.0p-53 * 2.0 - 1.0);
    }
}

__global__ void diff_kernel(const float* a, const float* b, int64_t n, double* out) {
    double num = 0, den = 0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double d = static_cast<double>(a[i]) - b[i];
        num += d * d;
        den += static_cast<double>(b[i]) * b[i];
    }
    atomicAdd(out, num);
    atomicAdd(out + 1, den);
}

}  // namespace
}  // namespace rcsg

using namespace rcsg;

extern "C" int rcsg_gemm_selftest(int64_t m, int64_t n, int64_t k, int64_t batch, int32_t gathered, int32_t iters,
                                  double* out_rel_err, double* out_ms_tc, double* out_ms_simt) {
    try {
        // A: [batch][m][k] (or [m*batch][k] folded), B: [batch or 1][n][k], C: [batch][m][n]
        const int64_t a_el = batch * m * k, b_el = (gathered ? batch : 1) * n * k, c_el = batch * m * n;
        float *a, *b, *c1, *c2;
        double* d;
        int32_t *ia, *ib, *fault;
        if (cudaMalloc(&a, 2 * a_el * 4) || cudaMalloc(&b, 2 * b_el * 4) || cudaMalloc(&c1, 2 * c_el * 4) ||
            cudaMalloc(&c2, 2 * c_el * 4) || cudaMalloc(&d, 16) || cudaMalloc(&ia, batch * 4) ||
            cudaMalloc(&ib, batch * 4) || cudaMalloc(&fault, 4))
            return RCSG_ERR_DEVICE;
        fill_rand<<<1024, 256>>>(a, 2 * a_el, 1);
        fill_rand<<<1024, 256>>>(b, 2 * b_el, 2);
        std::vector<int32_t> idx(batch);
        for (int64_t i = 0; i < batch; ++i) idx[i] = static_cast<int32_t>(i);
        cudaMemcpy(ia, idx.data(), batch * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(ib, idx.data(), batch * 4, cudaMemcpyHostToDevice);
        GemmArgs g{};
        g.a = a;
        g.a_plane = a_el;
        g.b = b;
        g.b_plane = b_el;
        g.k = k;
        g.n = n;
        g.fault = fault;
        if (gathered) {
            g.m = m;
            g.batch = batch;
            g.a_batch = m * k;
            g.b_batch = n * k;
            g.c_batch = m * n;
            g.ia = ia;
            g.ib = ib;
        } else {
            g.m = m * batch;
            g.batch = 1;
        }
        g.c_plane = c_el;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        float ms_tc = 0, ms_simt = 0;
        g.c = c1;
        const bool tc = gemm_tc_supported(g);
        if (tc) {
            launch_gemm_tc(g, 0, 0);
            cudaEventRecord(e0);
            for (int i = 0; i < iters; ++i) launch_gemm_tc(g, 0, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms_tc, e0, e1);
        }
        g.c = c2;
        launch_gemm_simt<float>(g, 0);
        cudaEventRecord(e0);
        for (int i = 0; i < std::max(1, iters / 4); ++i) launch_gemm_simt<float>(g, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms_simt, e0, e1);
        cudaMemset(d, 0, 16);
        if (tc) diff_kernel<<<1024, 256>>>(c1, c2, 2 * c_el, d);
        double h[2] = {0, 1};
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        const cudaError_t err = cudaGetLastError();
        *out_rel_err = tc ? std::sqrt(h[0] / h[1]) : -1.0;
        *out_ms_tc = tc ? ms_tc / iters : -1.0;
        *out_ms_simt = ms_simt / std::max(1, iters / 4);
        cudaFree(a);
        cudaFree(b);
        cudaFree(c1);
        cudaFree(c2);
        cudaFree(d);
        cudaFree(ia);
        cudaFree(ib);
        cudaFree(fault);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        return err == cudaSuccess ? RCSG_OK : RCSG_ERR_DEVICE;
    } catch (...) {
        return RCSG_ERR_DEVICE;
    }
}

// fp16 complex GEMM timing with an explicit output scatter map (kernel tuning):
// C[m][n] (through the map) = A[m][k] B[n][k]^T; returns ms per launch.
template <typename T>
int gemm_bench(int elem, int64_t m, int64_t n, int64_t k, int32_t m_bits, int32_t n_bits, const int8_t* m_pos,
               const int8_t* n_pos, int32_t iters, double* out_ms);

extern "C" int rcsg_gemm_bench_f16(int64_t m, int64_t n, int64_t k, int32_t m_bits, int32_t n_bits,
                                   const int8_t* m_pos, const int8_t* n_pos, int32_t iters, double* out_ms) {
    return gemm_bench<__half>(2, m, n, k, m_bits, n_bits, m_pos, n_pos, iters, out_ms);
}

// fp32 storage, kind::tf32
extern "C" int rcsg_gemm_bench_tf32(int64_t m, int64_t n, int64_t k, int32_t m_bits, int32_t n_bits,
                                    const int8_t* m_pos, const int8_t* n_pos, int32_t iters, double* out_ms) {
    return gemm_bench<float>(0, m, n, k, m_bits, n_bits, m_pos, n_pos, iters, out_ms);
}

namespace rcsg {
namespace {
template <typename T>
__global__ void fill_half(T* p, int64_t n, uint64_t seed) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        uint64_t z = seed + (i + 1) * 0x9e3779b97f4a7c15ull;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        z ^= z >> 31;
        store_c(p + i, static_cast<float>(static_cast<double>(z >> 11) * 0x1.0p-53 * 2.0 - 1.0));
    }
}
template <typename T>
__global__ void diff_half(const T* a, const T* b, int64_t n, double* out) {
    double num = 0, den = 0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double x = load_c(a + i), y = load_c(b + i);
        num += (x - y) * (x - y);
        den += y * y;
    }
    atomicAdd(out, num);
    atomicAdd(out + 1, den);
}
}  // namespace
}  // namespace rcsg

// 2-byte tensor-core GEMM vs the SIMT kernel of the same storage type on random operands, through an
// explicit output map (every epilogue kind / K-tile width); rel = ||TC-SIMT|| / ||SIMT||.
template <typename T>
int gemm_check(int elem, int64_t m, int64_t n, int64_t k, int32_t m_bits, int32_t n_bits, const int8_t* m_pos,
               const int8_t* n_pos, double* out_rel, int split_tf32 = 0) {
    try {
        T *a, *b, *c1, *c2;
        int32_t* fault;
        double* d;
        const int64_t c_el = m * n;
        constexpr int eb = sizeof(T);
        if (cudaMalloc(&a, 2 * m * k * eb) || cudaMalloc(&b, 2 * n * k * eb) || cudaMalloc(&c1, 2 * c_el * eb) ||
            cudaMalloc(&c2, 2 * c_el * eb) || cudaMalloc(&fault, 4) || cudaMalloc(&d, 16))
            return RCSG_ERR_DEVICE;
        fill_half<<<1024, 256>>>(a, 2 * m * k, 7);
        fill_half<<<1024, 256>>>(b, 2 * n * k, 9);
        cudaMemset(c1, 0, 2 * c_el * eb);
        cudaMemset(c2, 0, 2 * c_el * eb);
        GemmArgs g{};
        g.a = a;
        g.a_plane = m * k;
        g.b = b;
        g.b_plane = n * k;
        g.c_plane = c_el;
        g.m = m;
        g.n = n;
        g.k = k;
        g.batch = 1;
        g.fault = fault;
        g.scale_exp = eb == 2 ? -4 : 0;  // keep |C| well inside fp16
        g.om.m_bits = m_bits;
        g.om.n_bits = n_bits;
        g.om.scatter = m_bits + n_bits > 0;
        for (int j = 0; j < m_bits; ++j) g.om.m_pos[j] = m_pos[j];
        for (int j = 0; j < n_bits; ++j) g.om.n_pos[j] = n_pos[j];
        if (!gemm_tc_supported(g)) return RCSG_ERR_CONFIG;
        g.c = c1;
        g.split_tf32 = split_tf32;
        launch_gemm_tc(g, elem, 0);
        g.split_tf32 = 0;
        g.c = c2;
        launch_gemm_simt<T>(g, 0);
        cudaMemset(d, 0, 16);
        diff_half<<<1024, 256>>>(c1, c2, 2 * c_el, d);
        double h[2] = {0, 1};
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        const cudaError_t err = cudaGetLastError();
        *out_rel = std::sqrt(h[0] / h[1]);
        cudaFree(a);
        cudaFree(b);
        cudaFree(c1);
        cudaFree(c2);
        cudaFree(fault);
        cudaFree(d);
        return err == cudaSuccess ? RCSG_OK : RCSG_ERR_DEVICE;
    } catch (...) {
        return RCSG_ERR_DEVICE;
    }
}

extern "C" int rcsg_gemm_check_f16(int64_t m, int64_t n, int64_t k, int32_t m_bits, int32_t n_bits,
                                   const int8_t* m_pos, const int8_t* n_pos, double* out_rel) {
    return gemm_check<f16>(2, m, n, k, m_bits, n_bits, m_pos, n_pos, out_rel);
}

// the same check for bf16 operands (tcgen05 kind::f16 with BF16 inputs)
extern "C" int rcsg_gemm_check_bf16(int64_t m, int64_t n, int64_t k, int32_t m_bits, int32_t n_bits,
                                    const int8_t* m_pos, const int8_t* n_pos, double* out_rel) {
    return gemm_check<bf16>(1, m, n, k, m_bits, n_bits, m_pos, n_pos, out_rel);
}

// the same check for fp32 storage (tcgen05 kind::tf32 against the fp32 SIMT kernel)
extern "C" int rcsg_gemm_check_tf32(int64_t m, int64_t n, int64_t k, int32_t m_bits, int32_t n_bits,
                                    const int8_t* m_pos, const int8_t* n_pos, double* out_rel) {
    return gemm_check<float>(0, m, n, k, m_bits, n_bits, m_pos, n_pos, out_rel);
}

// split tf32 ("3xTF32": hi + lo fp32 operand halves on kind::tf32) against the fp32 SIMT kernel
extern "C" int rcsg_gemm_check_3xtf32(int64_t m, int64_t n, int64_t k, int32_t m_bits, int32_t n_bits,
                                      const int8_t* m_pos, const int8_t* n_pos, double* out_rel) {
    return gemm_check<float>(0, m, n, k, m_bits, n_bits, m_pos, n_pos, out_rel, 1);
}

// tcgen05 GEMM timing on random operands through an explicit output map (tools only)
template <typename T>
int gemm_bench(int elem, int64_t m, int64_t n, int64_t k, int32_t m_bits, int32_t n_bits, const int8_t* m_pos,
               const int8_t* n_pos, int32_t iters, double* out_ms) {
    try {
        T *a, *b, *c;
        int32_t* fault;
        constexpr int eb = sizeof(T);
        if (cudaMalloc(&a, 2 * m * k * eb) || cudaMalloc(&b, 2 * n * k * eb) || cudaMalloc(&c, 2 * m * n * eb) ||
            cudaMalloc(&fault, 4))
            return RCSG_ERR_DEVICE;
        rcsg::fill_half<<<1024, 256>>>(a, 2 * m * k, 7);
        rcsg::fill_half<<<1024, 256>>>(b, 2 * n * k, 9);
        GemmArgs g{};
        g.a = a;
        g.a_plane = m * k;
        g.b = b;
        g.b_plane = n * k;
        g.c = c;
        g.c_plane = m * n;
        g.m = m;
        g.n = n;
        g.k = k;
        g.batch = 1;
        g.fault = fault;
        g.scale_exp = eb == 2 ? -12 : 0;
        g.om.m_bits = m_bits;
        g.om.n_bits = n_bits;
        g.om.scatter = m_bits + n_bits > 0;
        for (int j = 0; j < m_bits; ++j) g.om.m_pos[j] = m_pos[j];
        for (int j = 0; j < n_bits; ++j) g.om.n_pos[j] = n_pos[j];
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        launch_gemm_tc(g, elem, 0);
        cudaEventRecord(e0);
        for (int i = 0; i < iters; ++i) launch_gemm_tc(g, elem, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        *out_ms = ms / iters;
        const cudaError_t err = cudaGetLastError();
        cudaFree(a);
        cudaFree(b);
        cudaFree(c);
        cudaFree(fault);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        return err == cudaSuccess ? RCSG_OK : RCSG_ERR_DEVICE;
    } catch (...) {
        return RCSG_ERR_DEVICE;
    }
}
