// Batched complex GEMV for contraction steps whose output has <= 4 columns (or
// rows): pure HBM streaming of the large operand, so no tensor cores.
//   C[v][m][n] = sum_k A[ia(v)][m][k] * B[ib(v)][n][k],  n <= 4  (or m <= 4)
// One warp per (variant, long row, k-split): 16-byte vector loads along K of
// both planes, the short operand's rows read through L1/L2, warp-shuffle
// reduction, partials written per split and summed in a fixed order
// (deterministic).  The reference computes these steps with the same ikj loop
// as every other step (contraction_engine.cpp:115-123).
#include <algorithm>

#include "kernels.cuh"

namespace rcsg {
namespace {

constexpr int kWarps = 8;
constexpr int kMaxShort = 4;

template <typename R>
struct Vec4;
template <>
struct Vec4<float> {
    using T = float4;
};
template <>
struct Vec4<double> {
    using T = double2;  // 16 B
};

template <typename R>
__global__ void __launch_bounds__(kWarps * 32)
    gemv_kernel(const GemmArgs g, int64_t rows, int shorts, int long_is_a, int64_t k_chunk, int splits, R* ws,
                int64_t ws_split) {
    using V = typename Vec4<R>::T;
    constexpr int kVec = sizeof(V) / sizeof(R);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t total = g.batch * rows * splits;
    for (int64_t w = static_cast<int64_t>(blockIdx.x) * kWarps + warp; w < total;
         w += static_cast<int64_t>(gridDim.x) * kWarps) {
        const int split = static_cast<int>(w % splits);
        const int64_t t = w / splits;
        const int64_t row = t % rows;
        const int64_t v = t / rows;
        const int64_t av = g.ia ? g.ia[v] : (g.a_batch ? v : 0);
        const int64_t bv = g.ib ? g.ib[v] : (g.b_batch ? v : 0);
        const R* A = static_cast<const R*>(g.a) + av * g.a_batch;
        const R* B = static_cast<const R*>(g.b) + bv * g.b_batch;
        // long operand row `row`, short operand rows 0..shorts-1
        const R* L = long_is_a ? A + row * g.k : B + row * g.k;
        const int64_t lplane = long_is_a ? g.a_plane : g.b_plane;
        const R* S = long_is_a ? B : A;
        const int64_t splane = long_is_a ? g.b_plane : g.a_plane;
        R acc_re[kMaxShort], acc_im[kMaxShort];
#pragma unroll
        for (int j = 0; j < kMaxShort; ++j) acc_re[j] = acc_im[j] = R(0);
        const int64_t k0 = split * k_chunk, k1 = min(g.k, k0 + k_chunk);
        if ((g.k % kVec) == 0) {
            for (int64_t kk = k0 + lane * kVec; kk < k1; kk += 32 * kVec) {
                const V lr = *reinterpret_cast<const V*>(L + kk);
                const V li = *reinterpret_cast<const V*>(L + lplane + kk);
                const R* lrp = reinterpret_cast<const R*>(&lr);
                const R* lip = reinterpret_cast<const R*>(&li);
#pragma unroll
                for (int j = 0; j < kMaxShort; ++j) {
                    if (j >= shorts) break;
                    const V sr = __ldg(reinterpret_cast<const V*>(S + j * g.k + kk));
                    const V si = __ldg(reinterpret_cast<const V*>(S + splane + j * g.k + kk));
                    const R* srp = reinterpret_cast<const R*>(&sr);
                    const R* sip = reinterpret_cast<const R*>(&si);
#pragma unroll
                    for (int e = 0; e < kVec; ++e) {
                        acc_re[j] = fma(lrp[e], srp[e], acc_re[j]);
                        acc_re[j] = fma(-lip[e], sip[e], acc_re[j]);
                        acc_im[j] = fma(lrp[e], sip[e], acc_im[j]);
                        acc_im[j] = fma(lip[e], srp[e], acc_im[j]);
                    }
                }
            }
        } else {
            for (int64_t kk = k0 + lane; kk < k1; kk += 32) {
                const R lr = L[kk], li = L[lplane + kk];
                for (int j = 0; j < shorts; ++j) {
                    const R sr = S[j * g.k + kk], si = S[splane + j * g.k + kk];
                    acc_re[j] = fma(lr, sr, acc_re[j]);
                    acc_re[j] = fma(-li, si, acc_re[j]);
                    acc_im[j] = fma(lr, si, acc_im[j]);
                    acc_im[j] = fma(li, sr, acc_im[j]);
                }
            }
        }
#pragma unroll
        for (int j = 0; j < kMaxShort; ++j)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                acc_re[j] += __shfl_xor_sync(0xffffffffu, acc_re[j], o);
                acc_im[j] += __shfl_xor_sync(0xffffffffu, acc_im[j], o);
            }
        if (lane == 0) {
            // C[v][m][n]: long rows are m when A is long, n otherwise
            for (int j = 0; j < shorts; ++j) {
                const int64_t mi = long_is_a ? row : j, ni = long_is_a ? j : row;
                const int64_t o = v * g.m * g.n + mi * g.n + ni;
                if (splits == 1) {
                    R* C = static_cast<R*>(g.c) + v * g.c_batch + out_row_off(g.om, g.n, mi) + out_col_off(g.om, ni);
                    C[0] = acc_re[j];
                    C[g.c_plane] = acc_im[j];
                    if (g.fault && (!isfinite(acc_re[j]) || !isfinite(acc_im[j]))) atomicMin(g.fault, g.step);
                } else {
                    ws[split * ws_split + o] = acc_re[j];
                    ws[split * ws_split + ws_split / 2 + o] = acc_im[j];
                }
            }
        }
    }
}

}  // namespace

bool gemv_supported(const GemmArgs& g) {
    return (g.n <= kMaxShort || g.m <= kMaxShort) && g.k >= 256;
}

template <typename R>
void launch_gemv(const GemmArgs& g, cudaStream_t st) {
    const bool long_is_a = g.n <= kMaxShort && (g.m > kMaxShort || g.m >= g.n);
    const int64_t rows = long_is_a ? g.m : g.n;
    const int shorts = static_cast<int>(long_is_a ? g.n : g.m);
    // k-splits so that every warp streams >= 2048 elements and the grid has >= 8 warps per SM
    int splits = 1;
    while (g.batch * rows * splits < 148 * 64 && g.k / (splits * 2) >= 2048) splits *= 2;
    const int64_t k_chunk = (g.k + splits - 1) / splits;
    R* ws = nullptr;
    int64_t ws_split = 0;
    if (splits > 1) {
        ws_split = 2 * g.batch * g.m * g.n;
        ws = static_cast<R*>(device_workspace(static_cast<size_t>(splits) * ws_split * sizeof(R), st));
    }
    const int64_t warps = g.batch * rows * splits;
    const int grid = static_cast<int>(std::min<int64_t>((warps + kWarps - 1) / kWarps, 148 * 64));
    gemv_kernel<R><<<grid, kWarps * 32, 0, st>>>(g, rows, shorts, long_is_a ? 1 : 0, k_chunk, splits, ws, ws_split);
    if (splits > 1) launch_splitk_reduce<R>(ws, ws_split, splits, g, st);
}
template void launch_gemv<float>(const GemmArgs&, cudaStream_t);
template void launch_gemv<double>(const GemmArgs&, cudaStream_t);

}  // namespace rcsg
