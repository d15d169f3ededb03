// Bit-permutation transpose of [V][2^rank] planar complex tensors — the
// "permute" of TTGT (reference contraction_engine.cpp:55-73, O(rank) index
// arithmetic per element on one core) as an HBM-bound shared-memory tiled
// transpose.  A tile is the set U of index bits made of the input's lowest bits
// and the sources of the output's lowest bits (up to 2^11 elements); every CTA
// reads its tiles along input-contiguous runs and writes along output-contiguous
// runs with 16-byte vectors.  Shared memory is XOR-swizzled so that gathers with
// any power-of-two stride are (at worst 2-way) conflict free.
#include <algorithm>
#include <stdexcept>
#include <vector>

#include "kernels.cuh"

namespace rcsg {

PermuteDesc make_permute(int rank, const int* src_bit) {
    if (rank > kMaxRank) throw std::runtime_error("tensor rank exceeds kMaxRank");
    PermuteDesc d{};
    d.rank = rank;
    std::vector<int> dst_of(rank);
    for (int q = 0; q < rank; ++q) dst_of[src_bit[q]] = q;
    std::vector<char> inU(rank, 0);
    int nU = 0, lo_in = 0, lo_out = 0;
    const int cap = std::min(kPermTileBits, rank);
    auto take = [&](int pos) {
        if (inU[pos]) return true;
        if (nU >= cap) return false;
        inU[pos] = 1;
        ++nU;
        return true;
    };
    // grow the tile alternately along the input's and the output's fastest bits;
    // bits already inside the tile extend the contiguous runs for free
    for (bool progress = true; progress;) {
        progress = false;
        if (lo_in < rank && take(lo_in)) {
            ++lo_in;
            progress = true;
        }
        if (lo_out < rank && take(src_bit[lo_out])) {
            ++lo_out;
            progress = true;
        }
    }
    std::vector<int> U;  // e ordering: input position ascending
    for (int p = 0; p < rank; ++p)
        if (inU[p]) U.push_back(p);
    std::vector<int> e_of_pos(rank, -1);
    for (int j = 0; j < nU; ++j) e_of_pos[U[j]] = j;
    std::vector<int> F;  // f ordering: output positions 0..lo_out-1, then the rest of U
    for (int q = 0; q < lo_out; ++q) F.push_back(q);
    std::vector<int> rest;
    for (int p : U)
        if (dst_of[p] >= lo_out) rest.push_back(dst_of[p]);
    std::sort(rest.begin(), rest.end());
    F.insert(F.end(), rest.begin(), rest.end());
    d.tile_bits = nU;
    d.vec = (lo_in >= 2 && lo_out >= 2) ? 1 : 0;
    for (int x = 0; x < 64; ++x) {
        int64_t il = 0, ih = 0, ol = 0, oh = 0, el = 0, eh = 0;
        for (int b = 0; b < 6; ++b) {
            if (!((x >> b) & 1)) continue;
            if (b < 5 && b < nU) {
                il += int64_t{1} << U[b];
                ol += int64_t{1} << F[b];
                el += int64_t{1} << e_of_pos[src_bit[F[b]]];
            }
            if (b + 5 < nU) {
                ih += int64_t{1} << U[b + 5];
                oh += int64_t{1} << F[b + 5];
                eh += int64_t{1} << e_of_pos[src_bit[F[b + 5]]];
            }
        }
        if (x < 32) {
            d.in_lo[x] = static_cast<int32_t>(il);
            d.out_lo[x] = static_cast<int32_t>(ol);
            d.e_lo[x] = static_cast<int32_t>(el);
        }
        d.in_hi[x] = static_cast<int32_t>(ih);
        d.out_hi[x] = static_cast<int32_t>(oh);
        d.e_hi[x] = static_cast<int32_t>(eh);
    }
    int j = 0;
    for (int p = 0; p < rank; ++p)
        if (!inU[p]) {
            d.outer_in[j] = int64_t{1} << p;
            d.outer_out[j] = int64_t{1} << dst_of[p];
            ++j;
        }
    d.n_outer = j;
    return d;
}

namespace {

__device__ __forceinline__ int swz(int e) { return e ^ (((e >> 5) ^ (e >> 10)) & 31); }

template <typename R>
struct Vec;
template <>
struct Vec<float> {
    using T = float4;
    static constexpr int N = 4;
};
template <>
struct Vec<double> {
    using T = double2;
    static constexpr int N = 2;
};
template <>
struct Vec<bf16> {
    using T = uint2;  // 4 bf16, same run requirement as float
    static constexpr int N = 4;
};
template <>
struct Vec<f16> {
    using T = uint2;
    static constexpr int N = 4;
};

constexpr int kThreads = 256;

template <typename R>
__global__ void __launch_bounds__(kThreads) permute_kernel(const R* __restrict__ in, int64_t in_plane,
                                                           R* __restrict__ out, int64_t out_plane, int64_t n_var,
                                                           const PermuteDesc d) {
    pdl_enter();
    using V = typename Vec<R>::T;
    constexpr int VN = Vec<R>::N;
    __shared__ int32_t in_lo[32], in_hi[64], out_lo[32], out_hi[64], e_lo[32], e_hi[64];
    extern __shared__ __align__(16) unsigned char smem_raw[];
    R* s_re = reinterpret_cast<R*>(smem_raw);
    R* s_im = s_re + (1 << kPermTileBits);
    for (int i = threadIdx.x; i < 64; i += blockDim.x) {
        if (i < 32) {
            in_lo[i] = d.in_lo[i];
            out_lo[i] = d.out_lo[i];
            e_lo[i] = d.e_lo[i];
        }
        in_hi[i] = d.in_hi[i];
        out_hi[i] = d.out_hi[i];
        e_hi[i] = d.e_hi[i];
    }
    __syncthreads();
    const int64_t payload = int64_t{1} << d.rank;
    const int T = 1 << d.tile_bits;
    const int64_t outer = int64_t{1} << d.n_outer;
    const int64_t total = outer * n_var;
    for (int64_t cta = blockIdx.x; cta < total; cta += gridDim.x) {
        const int64_t v = cta >> d.n_outer;
        const int64_t c = cta & (outer - 1);
        int64_t bi = v * payload, bo = v * payload;
        for (int j = 0; j < d.n_outer; ++j)
            if ((c >> j) & 1) {
                bi += d.outer_in[j];
                bo += d.outer_out[j];
            }
        if (d.vec) {
            for (int q = threadIdx.x; q < T / VN; q += kThreads) {
                const int e0 = q * VN;
                const int64_t off = bi + in_lo[e0 & 31] + in_hi[e0 >> 5];
                const V r = *reinterpret_cast<const V*>(in + off);
                const V i = *reinterpret_cast<const V*>(in + in_plane + off);
                const R* rp = reinterpret_cast<const R*>(&r);
                const R* ip = reinterpret_cast<const R*>(&i);
#pragma unroll
                for (int t = 0; t < VN; ++t) {
                    s_re[swz(e0 + t)] = rp[t];
                    s_im[swz(e0 + t)] = ip[t];
                }
            }
            __syncthreads();
            for (int q = threadIdx.x; q < T / VN; q += kThreads) {
                const int f0 = q * VN;
                const int64_t off = bo + out_lo[f0 & 31] + out_hi[f0 >> 5];
                V r, i;
                R* rp = reinterpret_cast<R*>(&r);
                R* ip = reinterpret_cast<R*>(&i);
#pragma unroll
                for (int t = 0; t < VN; ++t) {
                    const int e = e_lo[(f0 + t) & 31] + e_hi[(f0 + t) >> 5];
                    rp[t] = s_re[swz(e)];
                    ip[t] = s_im[swz(e)];
                }
                *reinterpret_cast<V*>(out + off) = r;
                *reinterpret_cast<V*>(out + out_plane + off) = i;
            }
        } else {
            for (int e = threadIdx.x; e < T; e += kThreads) {
                const int64_t off = bi + in_lo[e & 31] + in_hi[e >> 5];
                s_re[swz(e)] = in[off];
                s_im[swz(e)] = in[in_plane + off];
            }
            __syncthreads();
            for (int f = threadIdx.x; f < T; f += kThreads) {
                const int e = e_lo[f & 31] + e_hi[f >> 5];
                const int64_t off = bo + out_lo[f & 31] + out_hi[f >> 5];
                out[off] = s_re[swz(e)];
                out[out_plane + off] = s_im[swz(e)];
            }
        }
        __syncthreads();
    }
}

}  // namespace

template <typename R>
void launch_permute(const R* in, int64_t in_plane, R* out, int64_t out_plane, int64_t n_var,
                    const PermuteDesc& d, cudaStream_t st) {
    const int64_t total = (int64_t{1} << d.n_outer) * n_var;
    const int grid = static_cast<int>(std::min<int64_t>(total, 148 * 8));
    const size_t smem = 2 * (size_t{1} << kPermTileBits) * sizeof(R);
    launch_pdl(permute_kernel<R>, dim3(grid), dim3(kThreads), smem, st, in, in_plane, out, out_plane, n_var, d);
}
template void launch_permute<float>(const float*, int64_t, float*, int64_t, int64_t, const PermuteDesc&,
                                    cudaStream_t);
template void launch_permute<double>(const double*, int64_t, double*, int64_t, int64_t, const PermuteDesc&,
                                     cudaStream_t);
template void launch_permute<bf16>(const bf16*, int64_t, bf16*, int64_t, int64_t, const PermuteDesc&, cudaStream_t);
template void launch_permute<f16>(const f16*, int64_t, f16*, int64_t, int64_t, const PermuteDesc&, cudaStream_t);

}  // namespace rcsg
