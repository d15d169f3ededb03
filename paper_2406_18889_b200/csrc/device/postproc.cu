// Post-processing on device amplitudes (reference sampling.cpp):
//   |a|^2 -> global top-k ordered by (prob desc, lexicographic asc)   (:82-114)
//   per-group inverse-CDF direct sampling                             (:116-145)
//   linear XEB over the ideal probabilities of the samples            (:62-73)
//
// Top-k is a threshold select, not a sort of every candidate:
//   1. two sampled histogram passes (1/32 - 1/256 of the groups) over the
//      order-preserving 64-bit key of the probability pick a threshold key
//      expected to keep ~1.05 k candidates (binade, then 2^-12 of a binade);
//   2. ONE streaming pass over all M * 2^l amplitudes (16 B each) appends
//      every candidate at or above the threshold to a compact buffer
//      (warp-aggregated atomics); the same pass can draw each group's direct
//      sample (one warp per group, sequential f64 CDF as in the reference);
//   3. the buffer (~k entries) is put in order: with 32-bit keys by buckets of
//      the kept key range, each bucket ranked by one warp on the exact
//      (prob desc, lexkey asc) order (bucket_rank_kernel); with 64-bit keys by
//      a radix sort and a tie pass over runs of equal keys;
//   4. the first k entries are mapped to bitstring indices.
// The selection is exact whatever the threshold: step 2 counts every
// candidate at or above it, and when fewer than k (or more than the buffer)
// were found the call falls back to sorting all candidates.  Scratch memory
// is pooled per device, so steady-state calls do not allocate.
//
// The SplitMix64 stream is counter-based: the g-th draw of Rng(seed) is
// mix(seed + (g+1)*gamma) (rng.hpp:14-22), so every group samples independently
// and still reproduces the reference's sequence bit for bit.
#include <cub/cub.cuh>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cmath>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "executor.hpp"
#include "kernels.cuh"
#include "postproc.hpp"

namespace rcsg {

#define CUDA_OK(x)                                                                      \
    do {                                                                                \
        cudaError_t e_ = (x);                                                           \
        if (e_ != cudaSuccess)                                                          \
            throw Failure{RCSG_ERR_DEVICE, std::string("CUDA: ") + cudaGetErrorString(e_) + \
                                               " at " #x};                              \
    } while (0)

namespace {

constexpr int kHistBins = 4096;
constexpr uint64_t kPadKey = 0x7fffffffffffffffull;  // sorts after every non-negative probability

struct MemberMap {
    int32_t n, l;
    int32_t low_open;       // open qubits are 0..l-1: index = fixed << l | i
    int32_t open_pos[64];   // qubit of open bit j
    int32_t fixed_pos[64];  // qubit of fixed bit b
};

__device__ __forceinline__ uint64_t member_index(const MemberMap& mm, uint64_t fixed, uint64_t i) {
    if (mm.low_open) return (fixed << mm.l) | i;
    uint64_t idx = 0;
    for (int j = 0; j < mm.l; ++j) idx |= ((i >> j) & 1ull) << mm.open_pos[j];
    for (int b = 0; b < mm.n - mm.l; ++b) idx |= ((fixed >> b) & 1ull) << mm.fixed_pos[b];
    return idx;
}

__device__ __forceinline__ uint64_t lex_key(uint64_t idx, int n) { return __brevll(idx) >> (64 - n); }

// Probability of candidate t: std::norm(a) = re*re + im*im, rounded like the
// reference's complex<double> (no fused multiply-add).
__device__ __forceinline__ double prob_at(const double* __restrict__ src, int from_amps, int64_t t) {
    if (!from_amps) return src[t];
    const double2 a = reinterpret_cast<const double2*>(src)[t];
    return __dadd_rn(__dmul_rn(a.x, a.x), __dmul_rn(a.y, a.y));
}

// Unsigned key whose ascending order is the numeric order of doubles, with
// -0.0 == +0.0 (the reference's operator> treats them as equal).
__device__ __forceinline__ uint64_t asc_key(double p) {
    if (p == 0.0) p = 0.0;
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(p));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// shared-memory staging slots of direct_scan_kernel (> one load round of 8 x 256)
constexpr unsigned kDirectStage = 3072;

// Sort key of a kept candidate (ascending = probability descending).  64-bit:
// the full descending key.  32-bit: the distance of the ascending key above the
// threshold, shifted so that probabilities up to 1 fit (distinct probabilities
// collide only within ~1e-8 relative), inverted; equal keys are re-ordered
// exactly by tie_fix_kernel.
template <typename K>
__device__ __forceinline__ K sort_key(double p, uint64_t thr) {
    const uint64_t a = asc_key(p);
    if constexpr (sizeof(K) == 8) {
        return ~a;
    } else {
        const uint64_t span = asc_key(1.0) - thr;
        const int sh = max(0, 64 - __clzll(static_cast<long long>(span | 1)) - 32);
        const uint64_t d = (a - thr) >> sh;
        return ~static_cast<K>(d > 0xffffffffull ? 0xffffffffull : d);
    }
}

__device__ __forceinline__ void flag_nan(double p, int* bad) {
    if (p != p) atomicExch(bad, 1);
}

// ---- 1. sampled histograms -------------------------------------------------
// level 0: bins = top 12 bits of the ascending key (sign + exponent: binades);
// level 1: inside binade `sel` (from sel[0]), the next 12 bits.  Samples every
// `stride`-th group.  The last block to finish picks the bin (no separate
// launch): suffix sums of the histogram (from the top bin down) find the
// highest bin whose suffix reaches `want` (sample units); level 0 writes the
// binade and the samples in binades above it, level 1 the threshold key.
__device__ void pick_threshold_block(const uint32_t* __restrict__ hist, int level, double want,
                                     uint32_t* __restrict__ sel, uint64_t* __restrict__ thr, double* part) {
    __shared__ int found;
    const uint32_t* h = hist + level * kHistBins;
    const double base = level ? static_cast<double>(sel[1]) : 0.0;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int per_t = kHistBins / nt;
    const int b0 = per_t * (nt - 1 - tid);  // thread tid owns bins [b0, b0 + per_t); thread 0 the top ones
    double local = 0;
    for (int j = 0; j < per_t; ++j) local += __ldcg(h + b0 + j);
    part[tid] = local;
    if (tid == 0) found = -1;
    __syncthreads();
    for (int off = 1; off < nt; off <<= 1) {  // inclusive scan over chunks, top first
        const double v = tid >= off ? part[tid - off] : 0.0;
        __syncthreads();
        part[tid] += v;
        __syncthreads();
    }
    const double above = base + (tid ? part[tid - 1] : 0.0);  // samples in bins >= b0 + per_t
    if (above < want && above + local >= want) {  // the one chunk where the running count crosses
        double c = above;
        for (int j = per_t - 1; j >= 0; --j) {
            const double hj = __ldcg(h + b0 + j);
            if (c + hj >= want) {
                found = b0 + j;
                break;
            }
            c += hj;
        }
    }
    __syncthreads();
    int b = found < 0 ? 0 : found;  // nothing reaches `want`: keep everything
    if (level == 0 && b < 0x800) b = 0x800;  // never below +0.0: negative probabilities take the full path
    if (b < b0 || b >= b0 + per_t) return;  // the owner of bin b writes
    if (level == 0) {
        double c = above;  // samples in bins above b
        for (int j = per_t - 1; b0 + j > b; --j) c += __ldcg(h + b0 + j);
        sel[0] = static_cast<uint32_t>(b);
        sel[1] = static_cast<uint32_t>(c);
    } else {
        thr[0] = (static_cast<uint64_t>(sel[0]) << 52) | (static_cast<uint64_t>(b) << 40);
    }
}

// The sample: runs of kSampleRun consecutive groups, one run in every
// kSampleRun * stride groups (contiguous reads; 1/stride of the groups)
constexpr int64_t kSampleRun = 32;
__host__ __device__ __forceinline__ int64_t sampled_groups(int64_t n_groups, int64_t stride) {
    const int64_t period = kSampleRun * stride, full = n_groups / period, rem = n_groups - full * period;
    return full * kSampleRun + (rem < kSampleRun ? rem : kSampleRun);
}

// hist: 2 x kHistBins bins, then one completion counter per level (zeroed by the caller)
__global__ void __launch_bounds__(512) sample_hist_kernel(const double* __restrict__ src, int from_amps,
                                                          int64_t n_groups, int l, int64_t stride, int level,
                                                          uint32_t* __restrict__ sel, uint32_t* __restrict__ hist,
                                                          int* __restrict__ bad, double want,
                                                          uint64_t* __restrict__ thr) {
    __shared__ uint32_t h[kHistBins];
    __shared__ double part[512];
    __shared__ bool last;
    for (int i = threadIdx.x; i < kHistBins; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const int64_t per = int64_t{1} << l;
    const int64_t n_s = sampled_groups(n_groups, stride);
    const int64_t n_el = n_s * per;
    const uint32_t sel0 = level ? __ldcg(sel) : 0;
    // U independent loads per thread in flight
    constexpr int U = 4;
    const int64_t gs = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t e0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e0 < n_el; e0 += U * gs) {
        double pv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t e = e0 + u * gs;
            const int64_t j = e >> l;  // sampled group ordinal -> group (runs of kSampleRun groups)
            const int64_t g = (j / kSampleRun) * kSampleRun * stride + (j % kSampleRun);
            pv[u] = e < n_el ? prob_at(src, from_amps, g * per + (e & (per - 1))) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const bool in = e0 + u * gs < n_el;
            if (in) flag_nan(pv[u], bad);
            const uint64_t k = asc_key(pv[u]);
            // warp-aggregated: the samples crowd into a few binades (level 0), so
            // lanes with the same bin add once
            uint32_t bin = level == 0 ? static_cast<uint32_t>(k >> 52)
                                      : (static_cast<uint32_t>(k >> 52) == sel0 ? static_cast<uint32_t>((k >> 40) & 0xfff)
                                                                                 : 0xffffffffu);
            if (!in) bin = 0xffffffffu;
            const unsigned peers = __match_any_sync(__activemask(), bin);
            if (bin != 0xffffffffu && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&h[bin], __popc(peers));
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kHistBins; i += blockDim.x)
        if (h[i]) atomicAdd(&hist[level * kHistBins + i], h[i]);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&hist[2 * kHistBins + level], 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    pick_threshold_block(hist, level, want, sel, thr, part);
}

// warp minimum of the kept keys, one atomic per warp (whole warp converged)
template <typename K>
__device__ __forceinline__ void publish_min(K v, K* out, int lane) {
    if constexpr (sizeof(K) == 4) {
        v = __reduce_min_sync(0xffffffffu, v);
    } else {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    }
    if (lane == 0 && out && v != ~K{0})
        atomicMin(reinterpret_cast<std::conditional_t<sizeof(K) == 4, unsigned, unsigned long long>*>(out), v);
}

// ---- 2. the streaming pass ----------------------------------------------------
// Every candidate with asc_key >= *thr is appended as (descending key, t): the
// full 64-bit key and index (K = V = uint64_t), or, when the candidate count
// fits 32 bits, the key's top 32 bits and a 32-bit index (half the bytes to
// sort; equal truncated keys are re-ordered exactly by the tie pass).
// DIRECT: also draws each group's direct sample (one warp per group).
template <bool DIRECT, typename K, typename V>
__global__ void __launch_bounds__(256) scan_kernel(const double* __restrict__ src, int from_amps,
                                                   int64_t n_groups, int l, const uint64_t* __restrict__ thr_p,
                                                   K* __restrict__ out_key, V* __restrict__ out_t,
                                                   unsigned long long* __restrict__ counter, uint64_t cap,
                                                   int* __restrict__ bad, const uint64_t* __restrict__ fixed,
                                                   MemberMap mm, uint64_t seed, uint64_t* __restrict__ direct_out,
                                                   unsigned long long* __restrict__ zero_group,
                                                   K* __restrict__ kmin_out) {
    // kept candidates are staged in shared memory (warp-aggregated shared
    // atomics) and flushed with ONE global atomic per ~1-2K entries: a global
    // atomic per warp would serialise on the single counter
    // (4 loads per thread in flight: 8, with 3K staging slots, measured slower)
    constexpr unsigned kStage = 2048;
    constexpr int U = 4;
    __shared__ K s_key[kStage];
    __shared__ V s_t[kStage];
    __shared__ unsigned s_cnt;
    __shared__ unsigned long long s_base;
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    const bool collect = thr_p != nullptr;
    const uint64_t thr = collect ? *thr_p : ~0ull;
    const int lane = threadIdx.x & 31;
    K kmin = ~K{0};  // smallest kept key (= largest probability)
    auto stage = [&](bool take, double p, int64_t t) {
        const unsigned mask = __ballot_sync(0xffffffffu, take);
        if (!mask) return;
        unsigned base = 0;
        if (lane == 0) base = atomicAdd(&s_cnt, static_cast<unsigned>(__popc(mask)));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (take) {
            const unsigned pos = base + __popc(mask & ((1u << lane) - 1));
            const K key = sort_key<K>(p, thr);
            s_key[pos] = key;
            s_t[pos] = static_cast<V>(t);
            kmin = min(kmin, key);
        }
    };
    auto publish_kmin = [&]() { publish_min<K>(kmin, kmin_out, lane); };
    // block-uniform: flush when fewer than `room` free slots remain (or always)
    auto flush = [&](unsigned room, bool force) {
        __syncthreads();
        const unsigned n = s_cnt;
        __syncthreads();
        if (n == 0 || (!force && n + room <= kStage)) return;
        if (threadIdx.x == 0) s_base = atomicAdd(counter, static_cast<unsigned long long>(n));
        __syncthreads();
        const unsigned long long b = s_base;
        for (unsigned i = threadIdx.x; i < n; i += blockDim.x)
            if (b + i < cap) {
                out_key[b + i] = s_key[i];
                out_t[b + i] = s_t[i];
            }
        __syncthreads();
        if (threadIdx.x == 0) s_cnt = 0;
        __syncthreads();
    };
    if (!DIRECT) {
        // flat grid-stride over candidates, U independent 16-B loads per thread in flight.
        // Kept entries go to a warp-private slice of the staging buffer, flushed by the
        // warp alone (one global atomic per ~100-250 entries): no block barriers, so a
        // warp waiting on its loads never stalls the others (blockDim = 256: 8 slices)
        constexpr unsigned kWarpStage = kStage / 8;
        const int64_t total = n_groups << l;
        const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
        K* w_key = s_key + (threadIdx.x >> 5) * kWarpStage;
        V* w_t = s_t + (threadIdx.x >> 5) * kWarpStage;
        unsigned wcnt = 0;  // warp-uniform
        auto wflush = [&]() {
            __syncwarp();
            unsigned long long b = 0;
            if (lane == 0 && wcnt) b = atomicAdd(counter, static_cast<unsigned long long>(wcnt));
            b = __shfl_sync(0xffffffffu, b, 0);
            for (unsigned i = lane; i < wcnt; i += 32)
                if (b + i < cap) {
                    out_key[b + i] = w_key[i];
                    out_t[b + i] = w_t[i];
                }
            __syncwarp();
            wcnt = 0;
        };
        for (int64_t t0 = blockIdx.x * static_cast<int64_t>(blockDim.x); t0 < total; t0 += U * stride) {
            double p[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t t = t0 + u * stride + threadIdx.x;
                p[u] = t < total ? prob_at(src, from_amps, t) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t t = t0 + u * stride + threadIdx.x;
                const bool in = t < total;
                if (in) flag_nan(p[u], bad);
                const bool take = in && asc_key(p[u]) >= thr;
                const unsigned mask = __ballot_sync(0xffffffffu, take);
                if (take) {
                    const unsigned pos = wcnt + __popc(mask & ((1u << lane) - 1));
                    const K key = sort_key<K>(p[u], thr);
                    w_key[pos] = key;
                    w_t[pos] = static_cast<V>(t);
                    kmin = min(kmin, key);
                }
                wcnt += __popc(mask);
            }
            if (wcnt + U * 32 > kWarpStage) wflush();
        }
        wflush();
        publish_kmin();
        return;
    }
    // one warp per group (8 groups per block iteration, block-uniform loops):
    // lanes read chunks of 32 consecutive candidates; lane 0 folds each chunk
    // sequentially (the reference's left-to-right f64 sum)
    const int64_t per = int64_t{1} << l;
    const int wpb = blockDim.x / 32;
    for (int64_t g0 = blockIdx.x * static_cast<int64_t>(wpb); g0 < n_groups;
         g0 += static_cast<int64_t>(gridDim.x) * wpb) {
        const int64_t g = g0 + threadIdx.x / 32;
        const bool valid = g < n_groups;
        double total = 0.0;
        for (int64_t c = 0; c < per; c += 32) {
            const int64_t i = c + lane;
            const bool in = valid && i < per;
            double p = 0.0;
            if (in) {
                p = prob_at(src, from_amps, g * per + i);
                flag_nan(p, bad);
            }
            if (collect) {
                stage(in && asc_key(p) >= thr, p, g * per + i);
                flush(blockDim.x, false);
            }
            const int cnt = static_cast<int>(per - c < 32 ? per - c : 32);
            for (int j = 0; j < cnt; ++j) total = __dadd_rn(total, __shfl_sync(0xffffffffu, p, j));
        }
        if (!valid) continue;
        if (!(total > 0.0)) {
            if (lane == 0) {
                atomicMin(zero_group, static_cast<unsigned long long>(g));
                direct_out[g] = 0;
            }
            continue;
        }
        uint64_t z = seed + static_cast<uint64_t>(g + 1) * 0x9e3779b97f4a7c15ull;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        z ^= z >> 31;
        double u = __dmul_rn(static_cast<double>(z >> 11) * 0x1.0p-53, total);
        int64_t pick = per - 1;
        bool done = false;
        for (int64_t c = 0; c < per && !done; c += 32) {
            const int64_t i = c + lane;
            const double p = i < per ? prob_at(src, from_amps, g * per + i) : 0.0;  // L1/L2 hit
            const int cnt = static_cast<int>(per - c < 32 ? per - c : 32);
            for (int j = 0; j < cnt; ++j) {
                u = __dsub_rn(u, __shfl_sync(0xffffffffu, p, j));
                if (u <= 0.0) {
                    pick = c + j;
                    done = true;
                    break;
                }
            }
        }
        if (lane == 0) direct_out[g] = member_index(mm, fixed[g], static_cast<uint64_t>(pick));
    }
    if (collect) flush(0, true);
    publish_kmin();
}

// Direct sampling fused with the threshold pass, for groups of <= 8192
// candidates: each block iteration loads GPB whole groups (16-B amplitude
// loads, coalesced, many in flight) into a shared-memory probability tile,
// staging kept top-k candidates on the way (one flush check per load round);
// then thread g walks group g's row from shared memory.
//
// The reference draws u = r * total with total the left-to-right f64 sum, then
// subtracts the probabilities left to right until u <= 0 (sampling.cpp).  The
// walk keeps the left-to-right total bit for bit (one sequential pass that
// leaves the running sums s_i in the row) and finds the first s_i >= u by
// binary search.  The reference's running u_i differs from u - s_i by at most
// per * 2^-52 * total (+ an underflow term): when u lies farther than that
// from the two running sums around the crossing, the pick is the reference's;
// otherwise (probability ~1e-14 per group) the group re-runs the reference's
// exact subtraction chain from the amplitudes.
template <typename K, typename V>
__global__ void __launch_bounds__(256) direct_scan_kernel(const double* __restrict__ src, int from_amps,
                                                          int64_t n_groups, int l, int gpb,
                                                          const uint64_t* __restrict__ thr_p,
                                                          K* __restrict__ out_key, V* __restrict__ out_t,
                                                          unsigned long long* __restrict__ counter, uint64_t cap,
                                                          int* __restrict__ bad, const uint64_t* __restrict__ fixed,
                                                          MemberMap mm, uint64_t seed,
                                                          uint64_t* __restrict__ direct_out,
                                                          unsigned long long* __restrict__ zero_group,
                                                          double slack_mul, K* __restrict__ kmin_out) {
    extern __shared__ __align__(16) unsigned char dsm[];
    constexpr int U = 8;
    const unsigned stage_n = kDirectStage;
    K* s_key = reinterpret_cast<K*>(dsm);
    V* s_t = reinterpret_cast<V*>(dsm + stage_n * sizeof(K));
    const int64_t per = int64_t{1} << l;
    const int pitch = static_cast<int>(per) + 1;  // odd pitch: threads walking rows hit distinct banks
    double* tile = reinterpret_cast<double*>(dsm + stage_n * (sizeof(K) + sizeof(V)));
    __shared__ unsigned s_cnt;
    __shared__ unsigned long long s_base;
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    const bool collect = thr_p != nullptr;
    const uint64_t thr = collect ? *thr_p : ~0ull;
    const int lane = threadIdx.x & 31;
    K kmin = ~K{0};  // smallest kept key (= largest probability)
    const int64_t tile_el = static_cast<int64_t>(gpb) * per;
    const int64_t total = n_groups * per;
    // block-uniform: flush the staged candidates when fewer than `room` slots remain (or always)
    auto flush = [&](unsigned room, bool force) {
        __syncthreads();
        const unsigned n = s_cnt;
        __syncthreads();
        if (n == 0 || (!force && n + room <= stage_n)) return;
        if (threadIdx.x == 0) s_base = atomicAdd(counter, static_cast<unsigned long long>(n));
        __syncthreads();
        const unsigned long long b0 = s_base;
        for (unsigned i = threadIdx.x; i < n; i += blockDim.x)
            if (b0 + i < cap) {
                out_key[b0 + i] = s_key[i];
                out_t[b0 + i] = s_t[i];
            }
        __syncthreads();
        if (threadIdx.x == 0) s_cnt = 0;
        __syncthreads();
    };
    // one load round: U independent 16-B loads per thread in flight
    auto load_round = [&](int64_t base_t, int64_t e0, double* pv) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t e = e0 + u * static_cast<int64_t>(blockDim.x) + threadIdx.x;
            pv[u] = (e < tile_el && base_t + e < total) ? prob_at(src, from_amps, base_t + e) : 0.0;
        }
    };
    // the round's probabilities into the tile, kept top-k candidates into the staging buffer
    auto consume_round = [&](int64_t base_t, int64_t e0, const double* pv) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t e = e0 + u * static_cast<int64_t>(blockDim.x) + threadIdx.x;
            const int64_t t = base_t + e;
            const bool in = e < tile_el && t < total;
            const double p = pv[u];
            if (in) {
                flag_nan(p, bad);
                tile[(e >> l) * pitch + (e & (per - 1))] = p;
            }
            if (collect) {
                const bool take = in && asc_key(p) >= thr;
                const unsigned mask = __ballot_sync(0xffffffffu, take);
                if (mask) {
                    unsigned b = 0;
                    if (lane == 0) b = atomicAdd(&s_cnt, static_cast<unsigned>(__popc(mask)));
                    b = __shfl_sync(0xffffffffu, b, 0);
                    if (take) {
                        const unsigned pos = b + __popc(mask & ((1u << lane) - 1));
                        const K key = sort_key<K>(p, thr);
                        s_key[pos] = key;
                        s_t[pos] = static_cast<V>(t);
                        kmin = min(kmin, key);
                    }
                }
            }
        }
    };
    // thread g walks group g0 + g of the tile
    auto walk = [&](int64_t g0) {
        const int64_t g = g0 + threadIdx.x;
        if (threadIdx.x < gpb && g < n_groups) {
            double* row = tile + threadIdx.x * pitch;
            double tot = 0.0;
            for (int64_t i = 0; i < per; ++i) {  // left-to-right total; the row keeps the running sums
                tot = __dadd_rn(tot, row[i]);
                row[i] = tot;
            }
            if (!(tot > 0.0)) {
                atomicMin(zero_group, static_cast<unsigned long long>(g));
                direct_out[g] = 0;
            } else {
                uint64_t z = seed + static_cast<uint64_t>(g + 1) * 0x9e3779b97f4a7c15ull;
                z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
                z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
                z ^= z >> 31;
                const double u = __dmul_rn(static_cast<double>(z >> 11) * 0x1.0p-53, tot);
                const double slack = slack_mul * static_cast<double>(per) * (tot * 0x1.0p-51 + 0x1.0p-1070);
                // first i with s_i >= u - slack (s is non-decreasing)
                int64_t lo = 0, hi = per - 1;
                while (lo < hi) {
                    const int64_t mid = (lo + hi) >> 1;
                    if (row[mid] >= u - slack) hi = mid;
                    else lo = mid + 1;
                }
                int64_t pick = lo;
                if (!(row[lo] >= u + slack)) {  // u near a running sum: the reference's exact chain
                    double w = u;
                    pick = per - 1;
                    for (int64_t i = 0; i < per; ++i) {
                        w = __dsub_rn(w, prob_at(src, from_amps, g * per + i));
                        if (w <= 0.0) {
                            pick = i;
                            break;
                        }
                    }
                }
                direct_out[g] = member_index(mm, fixed[g], static_cast<uint64_t>(pick));
            }
        }
    };
    if (tile_el <= U * static_cast<int64_t>(blockDim.x)) {
        // single-round tiles (gpb * 2^l <= U * 256): software pipeline - the next tile's
        // loads are in flight while this tile's groups are walked
        double pv[U];
        int64_t g0 = blockIdx.x * static_cast<int64_t>(gpb);
        if (g0 < n_groups) load_round(g0 * per, 0, pv);
        for (; g0 < n_groups; g0 += static_cast<int64_t>(gridDim.x) * gpb) {
            consume_round(g0 * per, 0, pv);
            if (collect) flush(U * blockDim.x, false);
            __syncthreads();
            const int64_t g1 = g0 + static_cast<int64_t>(gridDim.x) * gpb;
            if (g1 < n_groups) load_round(g1 * per, 0, pv);
            walk(g0);
            __syncthreads();  // the tile is reused
        }
    } else {
        for (int64_t g0 = blockIdx.x * static_cast<int64_t>(gpb); g0 < n_groups;
             g0 += static_cast<int64_t>(gridDim.x) * gpb) {
            const int64_t base_t = g0 * per;
            for (int64_t e0 = 0; e0 < tile_el; e0 += U * static_cast<int64_t>(blockDim.x)) {
                double pv[U];
                load_round(base_t, e0, pv);
                consume_round(base_t, e0, pv);
                if (collect) flush(U * blockDim.x, false);
            }
            __syncthreads();
            walk(g0);
            __syncthreads();  // the tile is reused
        }
    }
    if (collect) flush(0, true);
    publish_min<K>(kmin, kmin_out, lane);
}

// pad [count, cap) with the largest non-negative key; flags count < k or count > cap
template <typename K, typename V>
__global__ void pad_kernel(K* __restrict__ key, V* __restrict__ t, const unsigned long long* __restrict__ counter,
                           uint64_t cap, uint64_t k, int* __restrict__ fail) {
    const uint64_t cnt = *counter;
    if (blockIdx.x == 0 && threadIdx.x == 0 && (cnt < k || cnt > cap)) *fail = 1;
    const K pad = sizeof(K) == 8 ? static_cast<K>(kPadKey) : static_cast<K>(~K{0});  // sorts after every kept key
    for (uint64_t i = cnt + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < cap;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        key[i] = pad;
        t[i] = 0;
    }
}

// ---- 3. ties: runs of equal (possibly truncated) keys in the sorted prefix are
// re-ordered by (full descending key, lexicographic key) - the reference's
// (prob desc, lexkey asc) order
template <typename K, typename V>
__global__ void tie_fix_kernel(const K* __restrict__ key, V* __restrict__ t,
                               const unsigned long long* __restrict__ counter, uint64_t cap, uint64_t k,
                               const double* __restrict__ src, int from_amps, const uint64_t* __restrict__ fixed,
                               MemberMap mm, int* __restrict__ fail, uint64_t* __restrict__ out) {
    const uint64_t n = min(static_cast<uint64_t>(*counter), cap);  // real entries (pads excluded)
    const uint64_t low = (1ull << mm.l) - 1;
    auto order_key = [&](uint64_t ti, uint64_t& full, uint64_t& lex) {
        full = ~asc_key(prob_at(src, from_amps, static_cast<int64_t>(ti)));
        lex = lex_key(member_index(mm, fixed[ti >> mm.l], ti & low), mm.n);
    };
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < k;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (i > 0 && key[i] == key[i - 1]) continue;   // inside a run: its start writes it
        if (i + 1 >= n || key[i + 1] != key[i]) {      // run of one: the index straight out
            const uint64_t ti = t[i];
            out[i] = member_index(mm, fixed[ti >> mm.l], ti & low);
            continue;
        }
        uint64_t e = i + 1;
        while (e < n && key[e] == key[i] && e - i <= 256) ++e;
        if (e - i > 256) {  // pathological tie run: the caller sorts every candidate instead
            atomicExch(fail, 2);
            continue;
        }
        // (runs are re-ordered then written out below, up to k)
        // insertion sort of t[i, e) (runs are short)
        for (uint64_t a = i + 1; a < e; ++a) {
            const V ta = t[a];
            uint64_t fa, la;
            order_key(ta, fa, la);
            uint64_t b = a;
            while (b > i) {
                const V tb = t[b - 1];
                uint64_t fb, lb;
                order_key(tb, fb, lb);
                if (fb < fa || (fb == fa && lb <= la)) break;
                t[b] = tb;
                --b;
            }
            t[b] = ta;
        }
        for (uint64_t a = i; a < e && a < k; ++a) {
            const uint64_t ta = t[a];
            out[a] = member_index(mm, fixed[ta >> mm.l], ta & low);
        }
    }
}

// ---- 3'. bucket order: instead of radix-sorting every kept entry, the kept
// key range [largest probability, threshold] is cut into 2^18 buckets of
// equal width in the 64-bit descending key (bucket 0 = highest probabilities):
//   hist     counts per bucket (bcount, zeroed first), each entry keeping the
//            slot its atomic returned (its place inside the bucket);
//   scan     bstart = exclusive sum (cub), bstart[kBuckets] = total;
//   scatter  entries of buckets starting below k go to bucket start + slot
//            (key, candidate, bucket), no atomics;
//   rank     one thread per placed entry counts the entries of its bucket
//            ahead of it in (prob desc, lexkey asc, candidate position) order -
//            a strict total order: the exact key decides unless equal, so the
//            bitstring keys are computed only for ties - and writes its
//            bitstring index at bucket start + rank when that is below k.
// Buckets of more than kBucketMax entries (long runs of equal probabilities)
// take the full sort.  The scan pass writes the full 64-bit keys for this
// path, so nothing re-reads the amplitudes.
constexpr int kBucketBits = 18;
constexpr int kBuckets = 1 << kBucketBits;
constexpr uint32_t kBucketMax = 4096;

// keys lie in [kmin, ~thr]; shift so that the span fits kBucketBits
__device__ __forceinline__ int bucket_shift(uint64_t kmin, uint64_t thr) {
    const uint64_t span = ~thr - kmin;
    return max(0, 64 - __clzll(static_cast<long long>(span | 1)) - kBucketBits);
}

__global__ void bucket_hist_kernel(const uint64_t* __restrict__ key, const unsigned long long* __restrict__ counter,
                                   uint64_t cap, uint64_t k, const unsigned long long* __restrict__ kmin_p,
                                   const uint64_t* __restrict__ thr_p, uint32_t* __restrict__ bcount,
                                   uint32_t* __restrict__ rank_in, int* __restrict__ fail) {
    const uint64_t cnt = *counter;
    if (blockIdx.x == 0 && threadIdx.x == 0 && (cnt < k || cnt > cap)) *fail = 1;
    const uint64_t n = min(cnt, cap);
    const uint64_t kmin = *kmin_p;
    const int sh = bucket_shift(kmin, *thr_p);
    const uint64_t gs = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i0 = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i0 < n; i0 += 4 * gs) {
        uint64_t kk[4];  // 4 independent entries per thread in flight
#pragma unroll
        for (int u = 0; u < 4; ++u) kk[u] = i0 + u * gs < n ? key[i0 + u * gs] : 0;
        uint32_t rk[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)  // the entry's slot inside its bucket (any order)
            rk[u] = i0 + u * gs < n ? atomicAdd(&bcount[(kk[u] - kmin) >> sh], 1u) : 0u;
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (i0 + u * gs < n) rank_in[i0 + u * gs] = rk[u];
    }
}

template <typename V>
__global__ void bucket_scatter_kernel(const uint64_t* __restrict__ key, const V* __restrict__ t,
                                      const unsigned long long* __restrict__ counter, uint64_t cap, uint64_t k,
                                      const unsigned long long* __restrict__ kmin_p, const uint64_t* __restrict__ thr_p,
                                      const uint32_t* __restrict__ bstart, const uint32_t* __restrict__ rank_in,
                                      uint64_t* __restrict__ out_key, V* __restrict__ out_t,
                                      uint32_t* __restrict__ out_b) {
    const uint64_t n = min(static_cast<uint64_t>(*counter), cap);
    const uint64_t kmin = *kmin_p;
    const int sh = bucket_shift(kmin, *thr_p);
    const uint64_t gs = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i0 = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i0 < n; i0 += 4 * gs) {
        // 4 independent entries per thread in flight (key -> bucket start -> slot)
        uint64_t kk[4];
        uint32_t b[4], s0[4], pos[4];
        V tv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const bool in = i0 + u * gs < n;
            kk[u] = in ? key[i0 + u * gs] : kmin;
            tv[u] = in ? t[i0 + u * gs] : V{0};
            pos[u] = in ? rank_in[i0 + u * gs] : 0u;
            b[u] = static_cast<uint32_t>((kk[u] - kmin) >> sh);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            s0[u] = bstart[b[u]];
            pos[u] += s0[u];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (i0 + u * gs >= n || s0[u] >= k) continue;  // every rank of the bucket is >= k
            out_key[pos[u]] = kk[u];
            out_t[pos[u]] = tv[u];
            out_b[pos[u]] = b[u];
        }
    }
}

template <typename V>
__global__ void bucket_rank_kernel(const uint64_t* __restrict__ key, const V* __restrict__ t,
                                   const uint32_t* __restrict__ bid, const uint32_t* __restrict__ bstart,
                                   const unsigned long long* __restrict__ counter, uint64_t cap, uint64_t k,
                                   const uint64_t* __restrict__ fixed, MemberMap mm, int* __restrict__ fail,
                                   uint64_t* __restrict__ out) {
    const uint64_t n = min(static_cast<uint64_t>(*counter), cap);
    if (n < k) return;  // the call falls back to the full sort
    const uint64_t low = (1ull << mm.l) - 1;
    // positions >= k matter only inside the bucket that straddles k
    const uint64_t end = bstart[bid[k - 1] + 1];
    for (uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; p < end;
         p += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t b = bid[p];
        const uint32_t s0 = bstart[b], nb = bstart[b + 1] - s0;
        const V tp = t[p];
        if (nb > kBucketMax) {  // a long run of equal keys: full sort
            atomicExch(fail, 2);
            continue;
        }
        const uint64_t kp = key[p];
        uint32_t rank = 0, ties = 0;
        const uint32_t e = s0 + nb;
        uint32_t j = s0;
        for (; j + 4 <= e; j += 4) {  // 4 loads in flight
            const uint64_t k0 = key[j], k1 = key[j + 1], k2 = key[j + 2], k3 = key[j + 3];
            rank += (k0 < kp) + (k1 < kp) + (k2 < kp) + (k3 < kp);
            ties += (k0 == kp) + (k1 == kp) + (k2 == kp) + (k3 == kp);
        }
        for (; j < e; ++j) {
            const uint64_t kj = key[j];
            rank += kj < kp;
            ties += kj == kp;
        }
        if (ties > 1) {  // equal probabilities (besides itself): lexicographic key, then position
            const uint64_t lx = lex_key(member_index(mm, fixed[tp >> mm.l], tp & low), mm.n);
            for (j = s0; j < e; ++j) {
                if (key[j] != kp || j == p) continue;
                const V tj = t[j];
                const uint64_t lj = lex_key(member_index(mm, fixed[tj >> mm.l], tj & low), mm.n);
                rank += (lj < lx || (lj == lx && tj < tp)) ? 1u : 0u;
            }
        }
        if (s0 + rank < k) out[s0 + rank] = member_index(mm, fixed[tp >> mm.l], tp & low);
    }
}

// ---- 4. output indices
template <typename V>
__global__ void index_kernel(const V* __restrict__ t, uint64_t k, const uint64_t* __restrict__ fixed,
                             MemberMap mm, uint64_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < k;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t ti = t[i];
        out[i] = member_index(mm, fixed[ti >> mm.l], ti & ((1ull << mm.l) - 1));
    }
}

// ---- full path: every candidate keyed (lexkey sort, then stable prob sort)
__global__ void full_keys_kernel(const double* __restrict__ src, int from_amps, const uint64_t* __restrict__ fixed,
                                 MemberMap mm, int64_t total, uint64_t* __restrict__ lexk, uint64_t* __restrict__ t,
                                 int* __restrict__ bad) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t g = i >> mm.l;
        flag_nan(prob_at(src, from_amps, i), bad);
        lexk[i] = lex_key(member_index(mm, fixed[g], static_cast<uint64_t>(i & ((int64_t{1} << mm.l) - 1))), mm.n);
        t[i] = static_cast<uint64_t>(i);
    }
}

__global__ void gather_desc_kernel(const double* __restrict__ src, int from_amps, const uint64_t* __restrict__ t,
                                   int64_t n, uint64_t* __restrict__ key) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        key[i] = ~asc_key(prob_at(src, from_amps, static_cast<int64_t>(t[i])));
}

// ---- XEB: fixed-shape (deterministic) reduction of q over the samples
// q = |state[idx]|^2 from a device statevector, or q given per sample.
__global__ void xeb_kernel(const double* __restrict__ state, const double* __restrict__ q,
                           const uint64_t* __restrict__ idx, uint64_t count, double* __restrict__ out,
                           int* __restrict__ bad) {
    __shared__ double part[1024];
    double s = 0.0;
    for (uint64_t i = threadIdx.x; i < count; i += blockDim.x) {
        double v;
        if (state) {
            const double2 a = reinterpret_cast<const double2*>(state)[idx[i]];
            v = __dadd_rn(__dmul_rn(a.x, a.x), __dmul_rn(a.y, a.y));
        } else {
            v = q[i];
        }
        if (!(v >= 0.0) || isinf(v)) atomicExch(bad, 1);
        s += v;
    }
    part[threadIdx.x] = s;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = part[0];
}

MemberMap make_map(const rcsg_candidates& cs) {
    MemberMap mm{};
    if (cs.n_qubits < 1 || cs.n_qubits > 64 || cs.l < 0 || cs.l > cs.n_qubits)
        throw Failure{RCSG_ERR_CONFIG, "candidate set qubit counts out of range"};
    mm.n = cs.n_qubits;
    mm.l = cs.l;
    std::vector<char> is_open(cs.n_qubits, 0);
    for (int j = 0; j < cs.l; ++j) {
        const int q = cs.open_qubits[j];
        if (q < 0 || q >= cs.n_qubits || (j && q <= cs.open_qubits[j - 1]))
            throw Failure{RCSG_ERR_CONFIG, "open qubits must be distinct, ascending and in range"};
        mm.open_pos[j] = q;
        is_open[q] = 1;
    }
    int b = 0;
    for (int q = 0; q < cs.n_qubits; ++q)
        if (!is_open[q]) mm.fixed_pos[b++] = q;
    mm.low_open = 1;
    for (int j = 0; j < cs.l; ++j) mm.low_open &= cs.open_qubits[j] == j ? 1 : 0;
    return mm;
}

// Grow-only device scratch, pooled per (device, slot); post-processing calls
// on one device are serialised by the pool lock.
struct Pool {
    std::mutex mu;
    std::map<std::pair<int, int>, std::pair<void*, size_t>> bufs;
    std::map<int, cudaStream_t> streams;
    std::map<int, std::pair<cudaEvent_t, cudaEvent_t>> events;
};
Pool& pool() {
    static Pool* p = new Pool();  // never destroyed: buffers live until process exit
    return *p;
}
int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}
void* scratch(int slot, size_t bytes) {
    auto& e = pool().bufs[{current_device(), slot}];
    bytes = std::max<size_t>(bytes, 256);
    if (e.second < bytes) {
        if (e.first) cudaFree(e.first);
        e.first = nullptr;
        e.second = 0;
        CUDA_OK(cudaMalloc(&e.first, bytes));
        e.second = bytes;
    }
    return e.first;
}
template <class T>
T* scratch_as(int slot, size_t count) {
    return static_cast<T*>(scratch(slot, count * sizeof(T)));
}
cudaStream_t post_stream() {
    auto& s = pool().streams[current_device()];
    if (!s) CUDA_OK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    return s;
}

enum Slot {
    kFixed = 0, kKeyA, kKeyB, kTA, kTB, kTmp, kHist, kCounters, kOut, kDirect, kSel, kXeb, kBucket, kEnt, kBid, kRank
};

// per-bucket counts (kBuckets + 1, zeroed by each call) followed by the
// bucket starts (kBuckets + 1)
uint32_t* bucket_counts(cudaStream_t st) {
    const bool fresh = pool().bufs.count({current_device(), kBucket}) == 0;
    uint32_t* b = scratch_as<uint32_t>(kBucket, 2 * (kBuckets + 1));
    if (fresh) CUDA_OK(cudaMemsetAsync(b, 0, 2 * (kBuckets + 1) * sizeof(uint32_t), st));
    return b;
}

struct Counters {  // device-side control block
    unsigned long long count;
    unsigned long long zero_group;
    uint64_t thr;
    uint32_t sel[2];
    int bad;   // NaN probability seen
    int fail;  // fast path unusable
    int xbad;  // invalid ideal probability
    unsigned kmin;  // smallest kept 32-bit sort key
    unsigned long long kmin64;  // smallest kept 64-bit key (bucket range)
    double xsum[2];
};

template <typename K>
K* kmin_of(Counters* c) {
    if constexpr (sizeof(K) == 4) return reinterpret_cast<K*>(&c->kmin);
    else return reinterpret_cast<K*>(&c->kmin64);
}


int grid_for(int64_t work, int per_block) {
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((work + per_block - 1) / per_block, 148 * 8)));
}

// Exact (prob desc, lexkey asc) order of ALL candidates: stable radix sort by
// lexicographic key, then stable radix sort by the descending probability key.
void full_sort(const double* d_src, int from_amps, const MemberMap& mm, const uint64_t* d_fixed, int64_t total,
               Counters* d_ctl, cudaStream_t st, uint64_t** t_sorted) {
    uint64_t* ka = scratch_as<uint64_t>(kKeyA, total);
    uint64_t* kb = scratch_as<uint64_t>(kKeyB, total);
    uint64_t* ta = scratch_as<uint64_t>(kTA, total);
    uint64_t* tb = scratch_as<uint64_t>(kTB, total);
    full_keys_kernel<<<grid_for(total, 256), 256, 0, st>>>(d_src, from_amps, d_fixed, mm, total, ka, ta, &d_ctl->bad);
    size_t tmp1 = 0, tmp2 = 0;
    CUDA_OK(cub::DeviceRadixSort::SortPairs(nullptr, tmp1, ka, kb, ta, tb, total, 0, mm.n, st));
    CUDA_OK(cub::DeviceRadixSort::SortPairs(nullptr, tmp2, kb, ka, tb, ta, total, 0, 64, st));
    void* tmp = scratch(kTmp, std::max(tmp1, tmp2));
    CUDA_OK(cub::DeviceRadixSort::SortPairs(tmp, tmp1, ka, kb, ta, tb, total, 0, mm.n, st));
    gather_desc_kernel<<<grid_for(total, 256), 256, 0, st>>>(d_src, from_amps, tb, total, ka);
    CUDA_OK(cub::DeviceRadixSort::SortPairs(tmp, tmp2, ka, kb, tb, ta, total, 0, 64, st));
    *t_sorted = ta;
}

}  // namespace

PostResult postprocess(const rcsg_candidates& cs, const double* d_src, bool from_amps, uint64_t k,
                       uint64_t* out_top, bool want_direct, uint64_t seed, uint64_t* out_direct,
                       const double* d_state, bool device_out, int force_path) {
    std::lock_guard<std::mutex> lock(pool().mu);
    const MemberMap mm = make_map(cs);
    const int64_t G = static_cast<int64_t>(cs.n_groups);
    if (G < 1) throw Failure{RCSG_ERR_CONFIG, "candidate set has no groups"};
    const int64_t total = G << cs.l;
    if (out_top && (k < 1 || k > static_cast<uint64_t>(total)))
        throw Failure{RCSG_ERR_CONFIG, "top-k size k=" + std::to_string(k) + " outside [1, " +
                                           std::to_string(total) + "]"};
    if (!out_top) k = 0;
    cudaStream_t st = post_stream();
    auto& evp = pool().events[current_device()];
    if (!evp.first) {
        CUDA_OK(cudaEventCreate(&evp.first));
        CUDA_OK(cudaEventCreate(&evp.second));
    }
    uint64_t* d_fixed = scratch_as<uint64_t>(kFixed, G);
    CUDA_OK(cudaMemcpyAsync(d_fixed, cs.group_fixed, G * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
    Counters* d_ctl = scratch_as<Counters>(kCounters, 1);
    {
        const Counters init{0, ULLONG_MAX, 0, {0, 0}, 0, 0, 0, 0xffffffffu, ULLONG_MAX, {0, 0}};
        CUDA_OK(cudaMemcpyAsync(d_ctl, &init, sizeof(Counters), cudaMemcpyHostToDevice, st));
    }
    uint64_t* d_direct = want_direct ? scratch_as<uint64_t>(kDirect, G) : nullptr;
    uint64_t* d_top = out_top ? scratch_as<uint64_t>(kOut, k) : nullptr;
    // the caller's producers on the legacy default stream come first; the device
    // time (res.device_ms) starts once the candidate set is uploaded
    CUDA_OK(cudaEventRecord(evp.first, cudaStreamLegacy));
    CUDA_OK(cudaStreamWaitEvent(st, evp.first, 0));
    CUDA_OK(cudaEventRecord(evp.first, st));

    // threshold path for k well below the candidate count (force_path: 1 always, 2 never)
    // sample 1/stride of the groups: >= ~1024 expected top-k entries in the
    // sample keep the threshold tight (k / stride), 1/32 .. 1/256 of the groups
    const int64_t stride =
        total >= (int64_t{1} << 20) ? std::max<int64_t>(32, std::min<int64_t>(256, static_cast<int64_t>(k) / 1024)) : 1;
    bool fast = k > 0 && static_cast<double>(k) * 4 <= static_cast<double>(total) && force_path != 2;
    if (force_path == 1) fast = k > 0;
    const bool narrow = total <= (int64_t{1} << 32);  // 32-bit keys and indices in the compact buffer
    uint64_t cap = 0;
    void* keys = nullptr;
    void* ts = nullptr;
    if (fast) {
        const int64_t n_s = sampled_groups(G, stride);
        const double f = static_cast<double>(n_s) / static_cast<double>(G);  // sampled fraction
        const double c = static_cast<double>(k) * f;                          // expected samples in the top k
        const double want = c * 1.05 + 6.0 * std::sqrt(c) + 16.0;
        const double expect = want / f;
        cap = static_cast<uint64_t>(std::min<double>(static_cast<double>(total), 1.25 * expect + 4096.0));
        cap = std::max<uint64_t>(cap, k);
        uint32_t* hist = scratch_as<uint32_t>(kHist, 2 * kHistBins + 2);
        CUDA_OK(cudaMemsetAsync(hist, 0, (2 * kHistBins + 2) * sizeof(uint32_t), st));
        // few blocks: each merges its shared histogram into the global one with one atomic per bin
        const int hgrid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(((n_s << cs.l) + 4095) / 4096, 296)));
        for (int level = 0; level < 2; ++level) {
            sample_hist_kernel<<<hgrid, 512, 0, st>>>(d_src, from_amps, G, cs.l, stride, level, d_ctl->sel, hist,
                                                      &d_ctl->bad, want, &d_ctl->thr);
        }
        keys = scratch(kKeyA, cap * 8);
        ts = scratch(kTA, cap * 8);
    }
    auto scan = [&](auto kz, auto vz) {
        using K = decltype(kz);
        using V = decltype(vz);
        const uint64_t* thr = fast ? &d_ctl->thr : nullptr;
        K* kk = static_cast<K*>(keys);
        V* tt = static_cast<V*>(ts);
        if (want_direct && cs.l <= 13) {
            // shared-memory tile of gpb whole groups (<= 64 KB of probabilities)
            const int64_t per = int64_t{1} << cs.l;
            // 32 groups per tile (16.6 KB at l = 6): ~5 blocks per SM hide the load latency
            const int gpb = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(32, 8192 / per)));
            const size_t smem = kDirectStage * (sizeof(K) + sizeof(V)) + static_cast<size_t>(gpb) * (per + 1) * sizeof(double);
            static std::atomic<uint64_t> attr_done[3]{};  // per (K, V) instantiation
            if (first_on_device(attr_done[sizeof(K) == 4 ? 0 : (sizeof(V) == 8 ? 1 : 2)]))
                CUDA_OK(cudaFuncSetAttribute(direct_scan_kernel<K, V>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             160 * 1024));
            // RCSG_DIRECT_SLACK (test knob): widens the exactness margin so that
            // groups take the reference's subtraction chain
            const double slack_mul = getenv("RCSG_DIRECT_SLACK") ? atof(getenv("RCSG_DIRECT_SLACK")) : 1.0;
            // persistent grid: exactly the resident blocks (no partial last wave)
            int occ = 0, dev = 0, n_sm = 148;
            CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, direct_scan_kernel<K, V>, 256, smem));
            CUDA_OK(cudaGetDevice(&dev));
            CUDA_OK(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
            const int grid = static_cast<int>(
                std::max<int64_t>(1, std::min<int64_t>((G + gpb - 1) / gpb, static_cast<int64_t>(n_sm) * std::max(occ, 1))));
            direct_scan_kernel<K, V><<<grid, 256, smem, st>>>(d_src, from_amps, G, cs.l, gpb, thr, kk, tt,
                                                              &d_ctl->count, cap, &d_ctl->bad, d_fixed, mm, seed,
                                                              d_direct, &d_ctl->zero_group, slack_mul, kmin_of<K>(d_ctl));
        } else if (want_direct) {
            const int grid = grid_for(G, 8);  // 8 warps per block, one group per warp
            scan_kernel<true, K, V><<<grid, 256, 0, st>>>(d_src, from_amps, G, cs.l, thr, kk, tt, &d_ctl->count, cap,
                                                          &d_ctl->bad, d_fixed, mm, seed, d_direct,
                                                          &d_ctl->zero_group, kmin_of<K>(d_ctl));
        } else {
            scan_kernel<false, K, V><<<148 * 8, 256, 0, st>>>(d_src, from_amps, G, cs.l, thr, kk, tt, &d_ctl->count,
                                                              cap, &d_ctl->bad, d_fixed, mm, seed, d_direct,
                                                              &d_ctl->zero_group, kmin_of<K>(d_ctl));
        }
    };
    // bucket order (RCSG_TOPK_BUCKETS=0: the radix sort + tie pass instead):
    // the scan writes full 64-bit keys with 32-bit candidate indices
    const bool buckets = fast && narrow && !(getenv("RCSG_TOPK_BUCKETS") && atoi(getenv("RCSG_TOPK_BUCKETS")) == 0);
    if (fast || want_direct) {
        if (buckets) scan(uint64_t{0}, uint32_t{0});
        else if (narrow) scan(uint32_t{0}, uint32_t{0});
        else scan(uint64_t{0}, uint64_t{0});
    }
    auto select_buckets = [&]() {
        const uint64_t* ka = static_cast<const uint64_t*>(keys);
        const uint32_t* ta = static_cast<const uint32_t*>(ts);
        uint32_t* bcount = bucket_counts(st);
        uint32_t* bstart = bcount + (kBuckets + 1);
        uint64_t* kb = scratch_as<uint64_t>(kKeyB, cap);
        uint32_t* tb = scratch_as<uint32_t>(kTB, cap);
        uint32_t* bid = scratch_as<uint32_t>(kBid, cap);
        uint32_t* rk = scratch_as<uint32_t>(kRank, cap);
        CUDA_OK(cudaMemsetAsync(bcount, 0, (kBuckets + 1) * sizeof(uint32_t), st));
        size_t scan_bytes = 0;
        CUDA_OK(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, bcount, bstart, kBuckets + 1, st));
        void* scan_tmp = scratch(kTmp, scan_bytes);
        const int g = grid_for(static_cast<int64_t>(cap), 256);
        bucket_hist_kernel<<<g, 256, 0, st>>>(ka, &d_ctl->count, cap, k, &d_ctl->kmin64, &d_ctl->thr, bcount, rk,
                                              &d_ctl->fail);
        CUDA_OK(cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, bcount, bstart, kBuckets + 1, st));
        bucket_scatter_kernel<uint32_t><<<g, 256, 0, st>>>(ka, ta, &d_ctl->count, cap, k, &d_ctl->kmin64,
                                                           &d_ctl->thr, bstart, rk, kb, tb, bid);
        bucket_rank_kernel<uint32_t><<<g, 256, 0, st>>>(kb, tb, bid, bstart, &d_ctl->count, cap, k, d_fixed, mm,
                                                        &d_ctl->fail, d_top);
    };
    auto select_fast = [&](auto kz, auto vz) {
        using K = decltype(kz);
        using V = decltype(vz);
        K* ka = static_cast<K*>(keys);
        V* ta = static_cast<V*>(ts);
        pad_kernel<K, V><<<grid_for(static_cast<int64_t>(cap), 256), 256, 0, st>>>(ka, ta, &d_ctl->count, cap, k,
                                                                                 &d_ctl->fail);
        K* kb = static_cast<K*>(scratch(kKeyB, cap * sizeof(K)));
        V* tb = static_cast<V*>(scratch(kTB, cap * sizeof(V)));
        // 64-bit keys of non-negative probabilities have the top bit clear; 32-bit keys use every bit
        const int end_bit = sizeof(K) == 8 ? 63 : 32;
        size_t tmp_bytes = 0;
        CUDA_OK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, ka, kb, ta, tb, cap, 0, end_bit, st));
        void* tmp = scratch(kTmp, tmp_bytes);
        CUDA_OK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, ka, kb, ta, tb, cap, 0, end_bit, st));
        tie_fix_kernel<K, V><<<grid_for(static_cast<int64_t>(k), 256), 256, 0, st>>>(
            kb, tb, &d_ctl->count, cap, k, d_src, from_amps, d_fixed, mm, &d_ctl->fail, d_top);
    };
    auto select = [&](bool use_fast) {
        if (use_fast) {
            if (buckets) select_buckets();
            else if (narrow) select_fast(uint32_t{0}, uint32_t{0});
            else select_fast(uint64_t{0}, uint64_t{0});
        } else {
            uint64_t* t_sorted = nullptr;
            full_sort(d_src, from_amps, mm, d_fixed, total, d_ctl, st, &t_sorted);
            index_kernel<uint64_t><<<grid_for(static_cast<int64_t>(k), 256), 256, 0, st>>>(t_sorted, k, d_fixed, mm,
                                                                                         d_top);
        }
        if (d_state) xeb_kernel<<<1, 1024, 0, st>>>(d_state, nullptr, d_top, k, &d_ctl->xsum[0], &d_ctl->xbad);
    };
    if (out_top) select(fast);
    // XEB of the direct samples from the device statevector (ideal q)
    if (d_state && want_direct)
        xeb_kernel<<<1, 1024, 0, st>>>(d_state, nullptr, d_direct, G, &d_ctl->xsum[1], &d_ctl->xbad);
    CUDA_OK(cudaEventRecord(evp.second, st));
    Counters h{};
    CUDA_OK(cudaMemcpyAsync(&h, d_ctl, sizeof(Counters), cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
    PostResult res;
    res.fast_path = fast;
    res.candidates_kept = fast ? h.count : static_cast<uint64_t>(total);
    if (h.bad) throw Failure{RCSG_ERR_CONFIG, "probability is NaN"};
    if (want_direct && h.zero_group != ULLONG_MAX)
        throw Failure{RCSG_ERR_CONFIG,
                      "group " + std::to_string(h.zero_group) + " has zero total probability; cannot sample"};
    if (fast && h.fail) {  // threshold missed (or a long tie run): exact full sort instead
        res.fast_path = false;
        res.fallback = true;
        select(false);
        CUDA_OK(cudaEventRecord(evp.second, st));
        CUDA_OK(cudaMemcpyAsync(&h, d_ctl, sizeof(Counters), cudaMemcpyDeviceToHost, st));
        CUDA_OK(cudaStreamSynchronize(st));
    }
    float ms = 0.f;
    CUDA_OK(cudaEventElapsedTime(&ms, evp.first, evp.second));
    res.device_ms = ms;
    res.bytes = static_cast<uint64_t>(total) * (from_amps ? 16 : 8) + k * 8 + (want_direct ? G * 8 : 0);
    if (out_top)
        CUDA_OK(cudaMemcpyAsync(out_top, d_top, k * sizeof(uint64_t),
                                device_out ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    if (want_direct)
        CUDA_OK(cudaMemcpyAsync(out_direct, d_direct, G * sizeof(uint64_t),
                                device_out ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
    if (d_state) {
        if (h.xbad) throw Failure{RCSG_ERR_CONFIG, "missing or invalid ideal probability for a sample"};
        const double scale = std::ldexp(1.0, cs.n_qubits);
        if (out_top) res.xeb_top = scale * h.xsum[0] / static_cast<double>(k) - 1.0;
        if (want_direct) res.xeb_direct = scale * h.xsum[1] / static_cast<double>(G) - 1.0;
    }
    return res;
}

namespace {
int forced_path() {
    const char* e = getenv("RCSG_TOPK_PATH");  // tests: 1 threshold select, 2 full sort
    return e ? atoi(e) : 0;
}
}  // namespace

void topk_select(const rcsg_candidates& cs, const double* d_src, bool from_amps, uint64_t k, uint64_t* out,
                 cudaStream_t) {
    postprocess(cs, d_src, from_amps, k, out, false, 0, nullptr, nullptr, false, forced_path());
}

void direct_sample(const rcsg_candidates& cs, const double* d_src, bool from_amps, uint64_t seed, uint64_t* out,
                   cudaStream_t) {
    postprocess(cs, d_src, from_amps, 0, nullptr, true, seed, out, nullptr, false, 0);
}

double xeb_device(int n_qubits, uint64_t count, const double* d_state, const uint64_t* indices,
                  const double* d_q) {
    if (count == 0) throw Failure{RCSG_ERR_CONFIG, "XEB needs at least one sample"};
    std::lock_guard<std::mutex> lock(pool().mu);
    cudaStream_t st = post_stream();
    CUDA_OK(cudaStreamSynchronize(cudaStreamLegacy));
    Counters* d_ctl = scratch_as<Counters>(kCounters, 1);
    CUDA_OK(cudaMemsetAsync(d_ctl, 0, sizeof(Counters), st));
    const uint64_t* d_idx = nullptr;
    if (d_state) {
        uint64_t* di = scratch_as<uint64_t>(kXeb, count);
        CUDA_OK(cudaMemcpyAsync(di, indices, count * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
        d_idx = di;
    }
    xeb_kernel<<<1, 1024, 0, st>>>(d_state, d_q, d_idx, count, &d_ctl->xsum[0], &d_ctl->xbad);
    Counters h{};
    CUDA_OK(cudaMemcpyAsync(&h, d_ctl, sizeof(Counters), cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
    if (h.xbad) throw Failure{RCSG_ERR_CONFIG, "missing or invalid ideal probability for a sample"};
    return std::ldexp(1.0, n_qubits) * h.xsum[0] / static_cast<double>(count) - 1.0;
}

}  // namespace rcsg
