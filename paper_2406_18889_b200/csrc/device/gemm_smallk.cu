// Complex GEMM for steps with K <= 16 summed elements: these are outer-product
// like (output-write bound), so instead of tensor-core tiles each thread keeps
// one B row (K complex values) in registers and streams output rows, writing
// consecutive columns across the warp (128-B coalesced stores).
//   C[v][m][n] = sum_{k<K} A[ia(v)][m][k] * B[ib(v)][n][k]
#include <algorithm>

#include "kernels.cuh"

namespace rcsg {
namespace {

constexpr int kThreads = 256;
constexpr int kRows = 64;  // output rows per CTA

template <typename S, int K>
__global__ void __launch_bounds__(kThreads) smallk_kernel(const GemmArgs g, int nb, int rows) {
    pdl_enter();
    using R = typename Acc<S>::T;
    const R sc = pow2<R>(g.scale_exp);
    __shared__ R a_re[kRows][K], a_im[kRows][K];
    __shared__ int64_t row_off[kRows];
    // rows (<= kRows) output rows per tile: fewer for small grids, to spread them over the SMs
    const int64_t ntiles = (g.n + nb - 1) / nb, mtiles = (g.m + rows - 1) / rows;
    const int col = threadIdx.x % nb, rsub = threadIdx.x / nb, rstep = kThreads / nb;
    bool bad = false;
    for (int64_t tile = blockIdx.x; tile < g.batch * mtiles * ntiles; tile += gridDim.x) {
        const int64_t nt = tile % ntiles;
        const int64_t mt = (tile / ntiles) % mtiles;
        const int64_t v = tile / (ntiles * mtiles);
        const int64_t av = g.ia ? g.ia[v] : (g.a_batch ? v : 0);
        const int64_t bv = g.ib ? g.ib[v] : (g.b_batch ? v : 0);
        const S* A = static_cast<const S*>(g.a) + av * g.a_batch;
        const S* B = static_cast<const S*>(g.b) + bv * g.b_batch;
        S* C = static_cast<S*>(g.c) + v * g.c_batch;
        const int64_t m0 = mt * rows, n = nt * nb + col;
        __syncthreads();
        for (int e = threadIdx.x; e < rows * K; e += kThreads) {
            const int r = e / K, kk = e % K;
            const bool ok = m0 + r < g.m && kk < g.k;
            a_re[r][kk] = ok ? load_c(A + (m0 + r) * g.k + kk) : R(0);
            a_im[r][kk] = ok ? load_c(A + g.a_plane + (m0 + r) * g.k + kk) : R(0);
        }
        for (int r = threadIdx.x; r < rows; r += kThreads) row_off[r] = out_row_off(g.om, g.n, m0 + r);
        const int64_t col_off = out_col_off(g.om, n);
        R b_re[K], b_im[K];
#pragma unroll
        for (int kk = 0; kk < K; ++kk) {
            const bool ok = n < g.n && kk < g.k;
            b_re[kk] = ok ? load_c(B + n * g.k + kk) : R(0);
            b_im[kk] = ok ? load_c(B + g.b_plane + n * g.k + kk) : R(0);
        }
        __syncthreads();
        if (n < g.n) {
            for (int r = rsub; r < rows && m0 + r < g.m; r += rstep) {
                R cr = 0, ci = 0;
#pragma unroll
                for (int kk = 0; kk < K; ++kk) {
                    cr = fma(a_re[r][kk], b_re[kk], cr);
                    cr = fma(-a_im[r][kk], b_im[kk], cr);
                    ci = fma(a_re[r][kk], b_im[kk], ci);
                    ci = fma(a_im[r][kk], b_re[kk], ci);
                }
                const int64_t o = row_off[r] + col_off;
                cr = tf32_if(cr * sc, g.round_tf32);
                ci = tf32_if(ci * sc, g.round_tf32);
                store_c(C + o, cr);
                store_c(C + g.c_plane + o, ci);
                bad |= unstorable<S>(cr) || unstorable<S>(ci);
            }
        }
    }
    if (bad && g.fault) atomicMin(g.fault, g.step);
}

// Row mode, for outputs whose fastest bits come from the row index: one thread
// per row keeps its A row in registers; a CTA covers 256 rows x kColTile
// columns, the B tile is staged in shared memory (read as broadcasts) and
// consecutive threads store consecutive addresses.
constexpr int kColTile = 64;

template <typename S, int K>
__global__ void __launch_bounds__(kThreads) smallk_rows_kernel(const GemmArgs g) {
    pdl_enter();
    using R = typename Acc<S>::T;
    const R sc = pow2<R>(g.scale_exp);
    __shared__ R b_re[kColTile][K], b_im[kColTile][K];
    __shared__ int64_t col_off[kColTile];
    bool bad = false;
    const int64_t rtiles = (g.m + kThreads - 1) / kThreads, ctiles = (g.n + kColTile - 1) / kColTile;
    for (int64_t tile = blockIdx.x; tile < g.batch * rtiles * ctiles; tile += gridDim.x) {
        const int64_t ct = tile % ctiles;
        const int64_t rt = (tile / ctiles) % rtiles;
        const int64_t v = tile / (ctiles * rtiles);
        const int64_t av = g.ia ? g.ia[v] : (g.a_batch ? v : 0);
        const int64_t bv = g.ib ? g.ib[v] : (g.b_batch ? v : 0);
        const S* A = static_cast<const S*>(g.a) + av * g.a_batch;
        const S* B = static_cast<const S*>(g.b) + bv * g.b_batch;
        S* C = static_cast<S*>(g.c) + v * g.c_batch;
        const int64_t n0 = ct * kColTile, r = rt * kThreads + threadIdx.x;
        __syncthreads();
        for (int e = threadIdx.x; e < kColTile * K; e += kThreads) {
            const int c = e / K, kk = e % K;
            const bool ok = n0 + c < g.n && kk < g.k;
            b_re[c][kk] = ok ? load_c(B + (n0 + c) * g.k + kk) : R(0);
            b_im[c][kk] = ok ? load_c(B + g.b_plane + (n0 + c) * g.k + kk) : R(0);
        }
        for (int c = threadIdx.x; c < kColTile; c += kThreads) col_off[c] = out_col_off(g.om, n0 + c);
        __syncthreads();
        if (r >= g.m) continue;
        R a_re[K], a_im[K];
#pragma unroll
        for (int kk = 0; kk < K; ++kk) {
            const bool ok = kk < g.k;
            a_re[kk] = ok ? load_c(A + r * g.k + kk) : R(0);
            a_im[kk] = ok ? load_c(A + g.a_plane + r * g.k + kk) : R(0);
        }
        const int64_t roff = out_row_off(g.om, g.n, r);
        const int cend = static_cast<int>(g.n - n0 < kColTile ? g.n - n0 : kColTile);
#pragma unroll 4
        for (int c = 0; c < cend; ++c) {
            R cr = 0, ci = 0;
#pragma unroll
            for (int kk = 0; kk < K; ++kk) {
                cr = fma(a_re[kk], b_re[c][kk], cr);
                cr = fma(-a_im[kk], b_im[c][kk], cr);
                ci = fma(a_re[kk], b_im[c][kk], ci);
                ci = fma(a_im[kk], b_re[c][kk], ci);
            }
            const int64_t o = roff + col_off[c];
            cr = tf32_if(cr * sc, g.round_tf32);
            ci = tf32_if(ci * sc, g.round_tf32);
            store_c(C + o, cr);
            store_c(C + g.c_plane + o, ci);
            bad |= unstorable<S>(cr) || unstorable<S>(ci);
        }
    }
    if (bad && g.fault) atomicMin(g.fault, g.step);
}

template <typename R, int K>
void launch_k(const GemmArgs& g, cudaStream_t st) {
    if (g.om.scatter && g.om.m_bits >= 5 && g.om.m_pos[0] == 0 && g.om.m_pos[1] == 1) {
        const int64_t tiles = g.batch * ((g.m + kThreads - 1) / kThreads) * ((g.n + kColTile - 1) / kColTile);
        const int grid = static_cast<int>(std::min<int64_t>(tiles, 148 * 16));
        launch_pdl(smallk_rows_kernel<R, K>, dim3(std::max(grid, 1)), dim3(kThreads), 0, st, g);
        return;
    }
    const int nb = static_cast<int>(std::min<int64_t>(g.n, kThreads));
    const int64_t ntiles = g.batch * ((g.n + nb - 1) / nb);
    int rows = kRows;  // at least ~2 CTAs per SM when the problem allows
    while (rows > 4 && ntiles * ((g.m + rows - 1) / rows) < 296) rows /= 2;
    const int64_t tiles = ntiles * ((g.m + rows - 1) / rows);
    const int grid = static_cast<int>(std::min<int64_t>(tiles, 148 * 16));
    launch_pdl(smallk_kernel<R, K>, dim3(std::max(grid, 1)), dim3(kThreads), 0, st, g, nb, rows);
}

}  // namespace

bool gemm_smallk_supported(const GemmArgs& g) { return g.k <= 16; }

template <typename R>
void launch_gemm_smallk(const GemmArgs& g, cudaStream_t st) {
    if (g.k <= 1) launch_k<R, 1>(g, st);
    else if (g.k <= 2) launch_k<R, 2>(g, st);
    else if (g.k <= 4) launch_k<R, 4>(g, st);
    else if (g.k <= 8) launch_k<R, 8>(g, st);
    else launch_k<R, 16>(g, st);
}
template void launch_gemm_smallk<float>(const GemmArgs&, cudaStream_t);
template void launch_gemm_smallk<double>(const GemmArgs&, cudaStream_t);
template void launch_gemm_smallk<bf16>(const GemmArgs&, cudaStream_t);
template void launch_gemm_smallk<f16>(const GemmArgs&, cudaStream_t);

}  // namespace rcsg
