// Device kernels of the contraction path: leaf projection, bit-permutation
// transpose, SIMT complex GEMM, pass finalisation and compensated reduction.
// See kernels.cuh for the storage convention.
#include <algorithm>
#include <cstdio>
#include <stdexcept>
#include <map>
#include <mutex>
#include <vector>

#include "kernels.cuh"

namespace rcsg {

static inline int grid_cap() { return 148 * 16; }

// ------------------------------------------------------------------ leaves
// One CTA per leaf job; threads stride over (variant, element).
template <typename R>
__global__ void leaf_project_kernel(const LeafJob* __restrict__ jobs,
                                    const double* __restrict__ leaf_data,
                                    const uint64_t* __restrict__ codes,
                                    const PassSrc* __restrict__ pass_src,
                                    const PassState* __restrict__ state, R* __restrict__ arena,
                                    int round_tf32) {
    pdl_enter();
    const LeafJob j = jobs[blockIdx.x];
    const PassState ps = *state;
    // bits fixed by pass labels, and per-free-position source bit
    uint64_t fixed = 0;
    int free_src[kMaxLeafRank], free_obit[kMaxLeafRank];
    int nf = 0;
    for (int p = 0; p < j.rank; ++p) {
        const int bitpos = j.rank - 1 - p;
        if (j.kind[p] == 0) {
            free_src[nf] = bitpos;
            free_obit[nf++] = j.obit[p];
        } else if (j.kind[p] == 1) {
            const PassSrc s = pass_src[j.arg[p]];
            const int v = s.kind == 0 ? s.value
                                      : static_cast<int>(((s.kind == 1 ? ps.slice : ps.config) >> s.bit) & 1);
            fixed |= static_cast<uint64_t>(v) << bitpos;
        }
    }
    const int64_t payload = int64_t{1} << j.out_rank;
    const int64_t total = payload * j.n_var;
    for (int64_t t = threadIdx.x; t < total; t += blockDim.x) {
        const int64_t v = t / payload;
        const int64_t i = t - v * payload;
        uint64_t src = fixed;
        if (j.codes_off >= 0) {
            const uint64_t code = codes[j.codes_off + v];
            for (int p = 0; p < j.rank; ++p)
                if (j.kind[p] == 2) src |= ((code >> j.arg[p]) & 1) << (j.rank - 1 - p);
        }
        // free positions land on their planned output bits
        for (int q = 0; q < nf; ++q) src |= static_cast<uint64_t>((i >> free_obit[q]) & 1) << free_src[q];
        const double re = leaf_data[2 * (j.data_off + src)];
        const double im = leaf_data[2 * (j.data_off + src) + 1];
        using C = typename Acc<R>::T;
        store_c(arena + j.out_off + t, tf32_if(static_cast<C>(re), round_tf32));
        store_c(arena + j.out_off + j.out_plane + t, tf32_if(static_cast<C>(im), round_tf32));
    }
}

template <typename R>
void launch_leaf_project(const LeafJob* d_jobs, int n_jobs, const double* d_leaf_data,
                         const uint64_t* d_codes, const PassSrc* d_pass_src,
                         const PassState* d_state, R* arena, cudaStream_t st, int round_tf32) {
    if (n_jobs == 0) return;
    launch_pdl(leaf_project_kernel<R>, dim3(n_jobs), dim3(64), 0, st, d_jobs, d_leaf_data, d_codes, d_pass_src,
               d_state, arena, round_tf32);
}
template void launch_leaf_project<float>(const LeafJob*, int, const double*, const uint64_t*,
                                         const PassSrc*, const PassState*, float*, cudaStream_t, int);
template void launch_leaf_project<double>(const LeafJob*, int, const double*, const uint64_t*,
                                          const PassSrc*, const PassState*, double*, cudaStream_t, int);
template void launch_leaf_project<bf16>(const LeafJob*, int, const double*, const uint64_t*,
                                        const PassSrc*, const PassState*, bf16*, cudaStream_t, int);
template void launch_leaf_project<f16>(const LeafJob*, int, const double*, const uint64_t*,
                                       const PassSrc*, const PassState*, f16*, cudaStream_t, int);

// ------------------------------------------------------------------ SIMT GEMM
// 64x64 complex tile per CTA, 16x16 threads, 4x4 complex outputs per thread,
// K step 16.  Used for fp64 (reference-grade parity) and for shapes the
// tensor-core kernel does not cover (tiny m/n/k).
constexpr int BM = 64, BN = 64, BK = 16;

struct SplitK {
    int splits;
    int64_t k_chunk;
    void* ws;          // nullptr: write C directly
    int64_t ws_split;  // elements per split (both planes)
};

template <typename S>
__global__ void __launch_bounds__(256) gemm_simt_kernel(const GemmArgs g, const SplitK sk) {
    pdl_enter();
    using R = typename Acc<S>::T;
    __shared__ R As_re[BK][BM + 1], As_im[BK][BM + 1];
    __shared__ R Bs_re[BK][BN + 1], Bs_im[BK][BN + 1];
    const S* A = static_cast<const S*>(g.a);
    const S* B = static_cast<const S*>(g.b);
    S* Cm = static_cast<S*>(g.c);
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 16 + tx;
    const R sc = pow2<R>(g.scale_exp);
    const int64_t mt = (g.m + BM - 1) / BM, nt = (g.n + BN - 1) / BN;
    const int64_t tiles = mt * nt * g.batch * sk.splits;
    for (int64_t tile_s = blockIdx.x; tile_s < tiles; tile_s += gridDim.x) {
        const int split = static_cast<int>(tile_s % sk.splits);
        const int64_t tile = tile_s / sk.splits;
        const int64_t k_lo = split * sk.k_chunk, k_hi = min(g.k, k_lo + sk.k_chunk);
        const int64_t v = tile / (mt * nt);
        const int64_t rem = tile - v * mt * nt;
        const int64_t m0 = (rem / nt) * BM, n0 = (rem % nt) * BN;
        const int64_t av = g.ia ? g.ia[v] : (g.a_batch ? v : 0);
        const int64_t bv = g.ib ? g.ib[v] : (g.b_batch ? v : 0);
        const S* Ab = A + av * g.a_batch;
        const S* Bb = B + bv * g.b_batch;
        R acc_re[4][4], acc_im[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc_re[i][j] = acc_im[i][j] = R(0);
        for (int64_t k0 = k_lo; k0 < k_hi; k0 += BK) {
            // 64 rows x 16 k per operand: 1024 elements, 4 per thread
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int e = tid + r * 256;
                const int row = e >> 4, kk = e & 15;
                const int64_t gk = k0 + kk;
                R ar = 0, ai = 0, br = 0, bi = 0;
                if (gk < k_hi) {
                    if (m0 + row < g.m) {
                        const int64_t o = (m0 + row) * g.k + gk;
                        ar = load_c(Ab + o);
                        ai = load_c(Ab + g.a_plane + o);
                    }
                    if (n0 + row < g.n) {
                        const int64_t o = (n0 + row) * g.k + gk;
                        br = load_c(Bb + o);
                        bi = load_c(Bb + g.b_plane + o);
                    }
                }
                As_re[kk][row] = ar;
                As_im[kk][row] = ai;
                Bs_re[kk][row] = br;
                Bs_im[kk][row] = bi;
            }
            __syncthreads();
#pragma unroll
            for (int kk = 0; kk < BK; ++kk) {
                R a_r[4], a_i[4], b_r[4], b_i[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    a_r[i] = As_re[kk][ty + 16 * i];
                    a_i[i] = As_im[kk][ty + 16 * i];
                    b_r[i] = Bs_re[kk][tx + 16 * i];
                    b_i[i] = Bs_im[kk][tx + 16 * i];
                }
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        acc_re[i][j] = fma(a_r[i], b_r[j], acc_re[i][j]);
                        acc_re[i][j] = fma(-a_i[i], b_i[j], acc_re[i][j]);
                        acc_im[i][j] = fma(a_r[i], b_i[j], acc_im[i][j]);
                        acc_im[i][j] = fma(a_i[i], b_r[j], acc_im[i][j]);
                    }
            }
            __syncthreads();
        }
        R* W = sk.ws ? static_cast<R*>(sk.ws) + split * sk.ws_split + v * g.m * g.n : nullptr;
        S* Cb = Cm + v * g.c_batch;
        const int64_t wplane = g.batch * g.m * g.n;
        bool bad = false;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int64_t m = m0 + ty + 16 * i, n = n0 + tx + 16 * j;
                if (m < g.m && n < g.n) {
                    if (W) {
                        W[m * g.n + n] = acc_re[i][j];
                        W[wplane + m * g.n + n] = acc_im[i][j];
                        bad |= !isfinite(acc_re[i][j]) || !isfinite(acc_im[i][j]);
                    } else {
                        const int64_t o = out_row_off(g.om, g.n, m) + out_col_off(g.om, n);
                        const R vr = tf32_if(acc_re[i][j] * sc, g.round_tf32), vi = tf32_if(acc_im[i][j] * sc, g.round_tf32);
                        store_c(Cb + o, vr);
                        store_c(Cb + g.c_plane + o, vi);
                        bad |= unstorable<S>(vr) || unstorable<S>(vi);
                    }
                }
            }
        if (bad && g.fault && !sk.ws) atomicMin(g.fault, g.step);
    }
}

// Fixed-order split-K reduction shared by every GEMM kernel: C = sum_z W[z],
// W planar [plane][batch][m][n] per split, C written through the output map.
template <typename S>
__global__ void splitk_reduce_kernel(const typename Acc<S>::T* __restrict__ ws, int64_t ws_split, int splits,
                                     const GemmArgs g) {
    pdl_enter();
    using R = typename Acc<S>::T;
    const int64_t mn = g.m * g.n, per_plane = g.batch * mn;
    const R sc = pow2<R>(g.scale_exp);
    S* C = static_cast<S*>(g.c);
    bool bad = false;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < per_plane;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        R re = 0, im = 0;
        for (int z = 0; z < splits; ++z) {
            re += ws[z * ws_split + i];
            im += ws[z * ws_split + per_plane + i];
        }
        const int64_t v = i / mn, e = i - v * mn, mi = e / g.n, ni = e - mi * g.n;
        const int64_t o = v * g.c_batch + out_row_off(g.om, g.n, mi) + out_col_off(g.om, ni);
        re = tf32_if(re * sc, g.round_tf32);
        im = tf32_if(im * sc, g.round_tf32);
        store_c(C + o, re);
        store_c(C + g.c_plane + o, im);
        bad |= unstorable<S>(re) || unstorable<S>(im);
    }
    if (bad && g.fault) atomicMin(g.fault, g.step);
}

template <typename S>
void launch_splitk_reduce(const typename Acc<S>::T* ws, int64_t ws_split, int splits, const GemmArgs& g,
                          cudaStream_t st) {
    const int64_t per_plane = g.batch * g.m * g.n;
    const int grid = static_cast<int>(std::min<int64_t>((per_plane + 255) / 256, 148 * 16));
    launch_pdl(splitk_reduce_kernel<S>, dim3(std::max(grid, 1)), dim3(256), 0, st, ws, ws_split, splits, g);
}
template void launch_splitk_reduce<float>(const float*, int64_t, int, const GemmArgs&, cudaStream_t);
template void launch_splitk_reduce<double>(const double*, int64_t, int, const GemmArgs&, cudaStream_t);
template void launch_splitk_reduce<bf16>(const float*, int64_t, int, const GemmArgs&, cudaStream_t);
template void launch_splitk_reduce<f16>(const float*, int64_t, int, const GemmArgs&, cudaStream_t);

template <typename S>
void launch_gemm_simt(const GemmArgs& g, cudaStream_t st) {
    using R = typename Acc<S>::T;
    dim3 block(16, 16);
    const int64_t tiles = ((g.m + BM - 1) / BM) * ((g.n + BN - 1) / BN) * g.batch;
    // split long K loops until the grid covers two waves (deterministic reduction)
    SplitK sk{1, g.k, nullptr, 0};
    while (tiles * sk.splits < 296 && g.k / (sk.splits * 2) >= 256) sk.splits *= 2;
    if (sk.splits > 1) {
        sk.k_chunk = (g.k + sk.splits - 1) / sk.splits;
        sk.ws_split = 2 * g.batch * g.m * g.n;
        sk.ws = device_workspace(static_cast<size_t>(sk.splits) * sk.ws_split * sizeof(R), st);
    }
    const int grid = static_cast<int>(std::min<int64_t>(tiles * sk.splits, 148 * 32));
    launch_pdl(gemm_simt_kernel<S>, dim3(grid), block, 0, st, g, sk);
    if (sk.splits > 1) launch_splitk_reduce<S>(static_cast<const R*>(sk.ws), sk.ws_split, sk.splits, g, st);
}

// ------------------------------------------------------------------ slice tables
__global__ void table_io_kernel(const TableJob* __restrict__ jobs, const PassState* __restrict__ state,
                                char* __restrict__ arena, int elem_bytes, int to_table) {
    pdl_enter();
    const TableJob j = jobs[blockIdx.y];
    uint64_t idx = 0;  // pext(slice, mask)
    int b = 0;
    for (uint64_t m = j.mask; m; m &= m - 1, ++b)
        if (state->slice & (m & (~m + 1))) idx |= uint64_t{1} << b;
    const int64_t n = j.payload * elem_bytes;  // bytes per plane
    char* node = arena + j.node_off * elem_bytes;
    char* slot = static_cast<char*>(j.table) + idx * 2 * n;
    const int64_t node_plane = j.node_plane * elem_bytes;
    const bool vec = (n & 15) == 0 && (node_plane & 15) == 0 &&
                     ((reinterpret_cast<uintptr_t>(node) | reinterpret_cast<uintptr_t>(slot)) & 15) == 0;
    for (int pl = 0; pl < 2; ++pl) {
        char* a = node + pl * node_plane;
        char* t = slot + pl * n;
        if (vec) {  // 16-B vectors
            uint4* a4 = reinterpret_cast<uint4*>(a);
            uint4* t4 = reinterpret_cast<uint4*>(t);
            for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n / 16;
                 i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
                if (to_table) t4[i] = a4[i];
                else a4[i] = t4[i];
            }
        } else {
            for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
                 i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
                if (to_table) t[i] = a[i];
                else a[i] = t[i];
            }
        }
    }
}
void launch_table_io(const TableJob* jobs, int n_jobs, const PassState* state, void* arena, int elem_bytes,
                     int to_table, cudaStream_t st) {
    if (n_jobs <= 0) return;
    launch_pdl(table_io_kernel, dim3(16, n_jobs), dim3(256), 0, st, jobs, state, static_cast<char*>(arena),
               elem_bytes, to_table);
}

namespace {
std::map<std::pair<cudaStream_t, int>, std::pair<void*, size_t>>& workspace_pool() {
    static std::map<std::pair<cudaStream_t, int>, std::pair<void*, size_t>> pool;
    return pool;
}
std::mutex& workspace_mu() {
    static std::mutex mu;
    return mu;
}
}  // namespace

void* device_workspace(size_t bytes, cudaStream_t st, int slot) {
    // one growing scratch buffer per (stream, slot) (launches on a stream are
    // ordered); Program's destructor releases the entries of its streams
    std::lock_guard<std::mutex> lock(workspace_mu());
    auto& e = workspace_pool()[{st, slot}];
    if (bytes > e.second) {
        if (e.first) {
            cudaStreamSynchronize(st);
            cudaFree(e.first);
        }
        e.first = nullptr;
        if (cudaMalloc(&e.first, bytes) != cudaSuccess) throw std::runtime_error("workspace allocation failed");
        e.second = bytes;
    }
    return e.first;
}

void release_workspace(cudaStream_t st) {
    std::lock_guard<std::mutex> lock(workspace_mu());
    auto& pool = workspace_pool();
    bool synced = false;
    for (auto it = pool.begin(); it != pool.end();) {
        if (it->first.first != st) {
            ++it;
            continue;
        }
        if (it->second.first) {
            if (!synced) cudaStreamSynchronize(st);
            synced = true;
            cudaFree(it->second.first);
        }
        it = pool.erase(it);
    }
}

bool first_on_device(std::atomic<uint64_t>& done) {
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = uint64_t{1} << (dev & 63);
    return (done.fetch_or(bit) & bit) == 0;
}
template void launch_gemm_simt<float>(const GemmArgs&, cudaStream_t);
template void launch_gemm_simt<double>(const GemmArgs&, cudaStream_t);
template void launch_gemm_simt<bf16>(const GemmArgs&, cudaStream_t);
template void launch_gemm_simt<f16>(const GemmArgs&, cudaStream_t);

// ------------------------------------------------------------------ finalize
template <typename R>
__global__ void finalize_kernel(const R* __restrict__ root, int64_t root_plane, double root_scale, int64_t payload,
                                int rank, const int32_t* __restrict__ src_bit, int n_fin,
                                const int32_t* __restrict__ fin_g, const int32_t* __restrict__ fin_off,
                                const int32_t* __restrict__ ent_vid, const int32_t* __restrict__ ent_lo,
                                const PassState* __restrict__ state, double* __restrict__ acc) {
    pdl_enter();
    const int64_t total = n_fin * payload;
    const uint32_t lo_b = state->lo_begin, lo_e = state->lo_end;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t f = t / payload;
        const int64_t i = t - f * payload;
        int64_t p = 0;
        for (int j = 0; j < rank; ++j) p |= ((i >> j) & 1) << src_bit[j];
        const int64_t g = fin_g[f];
        double re = acc[2 * (g * payload + i)], im = acc[2 * (g * payload + i) + 1];
        for (int e = fin_off[f]; e < fin_off[f + 1]; ++e) {  // slices ascending
            const uint32_t lo = static_cast<uint32_t>(ent_lo[e]);
            if (lo < lo_b || lo >= lo_e) continue;
            const int64_t o = static_cast<int64_t>(ent_vid[e]) * payload + p;
            re += static_cast<double>(load_c(root + o)) * root_scale;
            im += static_cast<double>(load_c(root + root_plane + o)) * root_scale;
        }
        acc[2 * (g * payload + i)] = re;
        acc[2 * (g * payload + i) + 1] = im;
    }
}

template <typename R>
void launch_finalize(const R* root, int64_t root_plane, double root_scale, int64_t payload, int rank,
                     const int32_t* d_src_bit_of_canon, int n_fin, const int32_t* d_fin_g, const int32_t* d_fin_off,
                     const int32_t* d_ent_vid, const int32_t* d_ent_lo, const PassState* d_state, double* acc,
                     cudaStream_t st) {
    const int64_t total = n_fin * payload;
    const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, grid_cap()));
    launch_pdl(finalize_kernel<R>, dim3(std::max(grid, 1)), dim3(256), 0, st, root, root_plane, root_scale, payload,
               rank, d_src_bit_of_canon, n_fin, d_fin_g, d_fin_off, d_ent_vid, d_ent_lo, d_state, acc);
}
#define RCSG_FIN(R)                                                                                               \
    template void launch_finalize<R>(const R*, int64_t, double, int64_t, int, const int32_t*, int, const int32_t*, \
                                     const int32_t*, const int32_t*, const int32_t*, const PassState*, double*,    \
                                     cudaStream_t);
RCSG_FIN(float)
RCSG_FIN(double)
RCSG_FIN(bf16)
RCSG_FIN(f16)
#undef RCSG_FIN

// ------------------------------------------------------------------ misc
__global__ void kahan_kernel(double* res, double* comp, const double* part, int64_t n) {
    pdl_enter();
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double y = part[i] - comp[i];
        const double s = __dadd_rn(res[i], y);
        comp[i] = __dsub_rn(__dsub_rn(s, res[i]), y);
        res[i] = s;
    }
}
void launch_kahan(double* res, double* comp, const double* part, int64_t n, cudaStream_t st) {
    const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, grid_cap()));
    launch_pdl(kahan_kernel, dim3(std::max(grid, 1)), dim3(256), 0, st, res, comp, part, n);
}

__global__ void maxabs_kernel(const float* buf, int64_t plane, int64_t count, float* out) {
    pdl_enter();
    float m = 0.f;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        m = fmaxf(m, fmaxf(fabsf(buf[i]), fabsf(buf[plane + i])));
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<int*>(out), __float_as_int(m));  // m >= 0
}
void launch_maxabs(const float* buf, int64_t plane, int64_t count, float* out, cudaStream_t st) {
    const int grid = static_cast<int>(std::min<int64_t>((count + 255) / 256, grid_cap()));
    launch_pdl(maxabs_kernel, dim3(std::max(grid, 1)), dim3(256), 0, st, buf, plane, count, out);
}

__global__ void fill_kernel(double* p, double v, int64_t n) {
    pdl_enter();
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        p[i] = v;
}
void launch_fill(double* p, double v, int64_t n, cudaStream_t st) {
    const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, grid_cap()));
    launch_pdl(fill_kernel, dim3(std::max(grid, 1)), dim3(256), 0, st, p, v, n);
}

__global__ void set_pass_kernel(PassState* s, uint64_t slice, uint64_t config, uint32_t lo_begin, uint32_t lo_end) {
    pdl_enter();
    s->slice = slice;
    s->config = config;
    s->lo_begin = lo_begin;
    s->lo_end = lo_end;
}
void launch_set_pass(PassState* d_state, uint64_t slice, uint64_t config, uint32_t lo_begin, uint32_t lo_end,
                     cudaStream_t st) {
    launch_pdl(set_pass_kernel, dim3(1), dim3(1), 0, st, d_state, slice, config, lo_begin, lo_end);
}

}  // namespace rcsg
