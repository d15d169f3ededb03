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

// 16-byte vector of storage elements
template <typename S>
struct Vec16;
template <>
struct Vec16<float> {
    using T = float4;
};
template <>
struct Vec16<double> {
    using T = double2;
};
template <>
struct Vec16<bf16> {
    using T = uint4;  // 8 bf16
};
template <>
struct Vec16<f16> {
    using T = uint4;  // 8 fp16
};

template <typename S>
__global__ void __launch_bounds__(kWarps * 32)
    gemv_kernel(const GemmArgs g, int64_t rows, int shorts, int long_is_a, int64_t k_chunk, int splits,
                typename Acc<S>::T* ws, int64_t ws_split) {
    pdl_enter();
    using R = typename Acc<S>::T;
    using V = typename Vec16<S>::T;
    constexpr int kVec = sizeof(V) / sizeof(S);
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
        const S* A = static_cast<const S*>(g.a) + av * g.a_batch;
        const S* B = static_cast<const S*>(g.b) + bv * g.b_batch;
        // long operand row `row`, short operand rows 0..shorts-1
        const S* L = long_is_a ? A + row * g.k : B + row * g.k;
        const int64_t lplane = long_is_a ? g.a_plane : g.b_plane;
        const S* Sh = long_is_a ? B : A;
        const int64_t splane = long_is_a ? g.b_plane : g.a_plane;
        R acc_re[kMaxShort], acc_im[kMaxShort];
#pragma unroll
        for (int j = 0; j < kMaxShort; ++j) acc_re[j] = acc_im[j] = R(0);
        const int64_t k0 = split * k_chunk, k1 = min(g.k, k0 + k_chunk);
        if ((g.k % kVec) == 0) {
            for (int64_t kk = k0 + lane * kVec; kk < k1; kk += 32 * kVec) {
                const V lr = *reinterpret_cast<const V*>(L + kk);
                const V li = *reinterpret_cast<const V*>(L + lplane + kk);
                const S* lrp = reinterpret_cast<const S*>(&lr);
                const S* lip = reinterpret_cast<const S*>(&li);
#pragma unroll
                for (int j = 0; j < kMaxShort; ++j) {
                    if (j >= shorts) break;
                    const V sr = __ldg(reinterpret_cast<const V*>(Sh + j * g.k + kk));
                    const V si = __ldg(reinterpret_cast<const V*>(Sh + splane + j * g.k + kk));
                    const S* srp = reinterpret_cast<const S*>(&sr);
                    const S* sip = reinterpret_cast<const S*>(&si);
#pragma unroll
                    for (int e = 0; e < kVec; ++e) {
                        const R a = load_c(lrp + e), b = load_c(lip + e), c = load_c(srp + e), d = load_c(sip + e);
                        acc_re[j] = fma(a, c, acc_re[j]);
                        acc_re[j] = fma(-b, d, acc_re[j]);
                        acc_im[j] = fma(a, d, acc_im[j]);
                        acc_im[j] = fma(b, c, acc_im[j]);
                    }
                }
            }
        } else {
            for (int64_t kk = k0 + lane; kk < k1; kk += 32) {
                const R lr = load_c(L + kk), li = load_c(L + lplane + kk);
                for (int j = 0; j < shorts; ++j) {
                    const R sr = load_c(Sh + j * g.k + kk), si = load_c(Sh + splane + j * g.k + kk);
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
                    S* C = static_cast<S*>(g.c) + v * g.c_batch + out_row_off(g.om, g.n, mi) + out_col_off(g.om, ni);
                    const R sc = pow2<R>(g.scale_exp), vr = tf32_if(acc_re[j] * sc, g.round_tf32),
                            vi = tf32_if(acc_im[j] * sc, g.round_tf32);
                    store_c(C, vr);
                    store_c(C + g.c_plane, vi);
                    if (g.fault && (unstorable<S>(vr) || unstorable<S>(vi))) atomicMin(g.fault, g.step);
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

template <typename S>
void launch_gemv(const GemmArgs& g, cudaStream_t st) {
    using R = typename Acc<S>::T;
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
    launch_pdl(gemv_kernel<S>, dim3(grid), dim3(kWarps * 32), 0, st, g, rows, shorts, long_is_a ? 1 : 0, k_chunk, splits, ws, ws_split);
    if (splits > 1) launch_splitk_reduce<S>(ws, ws_split, splits, g, st);
}
template void launch_gemv<float>(const GemmArgs&, cudaStream_t);
template void launch_gemv<double>(const GemmArgs&, cudaStream_t);
template void launch_gemv<bf16>(const GemmArgs&, cudaStream_t);
template void launch_gemv<f16>(const GemmArgs&, cudaStream_t);

}  // namespace rcsg
