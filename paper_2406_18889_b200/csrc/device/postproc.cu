// Post-processing on device amplitudes (reference sampling.cpp):
//   |a|^2 -> global top-k ordered by (prob desc, lexicographic asc)   (:82-114)
//   per-group inverse-CDF direct sampling                             (:116-145)
// The SplitMix64 stream is counter-based: the g-th draw of Rng(seed) is
// mix(seed + (g+1)*gamma) (rng.hpp:14-22), so every group samples independently
// on its own thread and still reproduces the reference's sequence bit for bit.
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <string>
#include <vector>

#include "executor.hpp"
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

struct MemberMap {
    int32_t n, l;
    int32_t open_pos[64];   // qubit of open bit j
    int32_t fixed_pos[64];  // qubit of fixed bit b
};

__device__ __forceinline__ uint64_t member_index(const MemberMap& mm, uint64_t fixed, uint64_t i) {
    uint64_t idx = 0;
    for (int j = 0; j < mm.l; ++j) idx |= ((i >> j) & 1ull) << mm.open_pos[j];
    for (int b = 0; b < mm.n - mm.l; ++b) idx |= ((fixed >> b) & 1ull) << mm.fixed_pos[b];
    return idx;
}

__device__ __forceinline__ uint64_t lex_key(uint64_t idx, int n) {
    return __brevll(idx) >> (64 - n);
}

// keys: lexicographic key (sorted first), then ~prob bits (sorted second, stable)
__global__ void topk_keys_kernel(const double* __restrict__ src, int from_amps, const uint64_t* __restrict__ fixed,
                                 MemberMap mm, int64_t total, uint64_t* __restrict__ lexk,
                                 uint64_t* __restrict__ probk, uint64_t* __restrict__ idx) {
    const int64_t per = int64_t{1} << mm.l;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t g = t / per, i = t - g * per;
        double p;
        if (from_amps) {
            const double re = src[2 * t], im = src[2 * t + 1];
            p = __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im));
        } else {
            p = src[t];
        }
        const uint64_t m = member_index(mm, fixed[g], static_cast<uint64_t>(i));
        lexk[t] = lex_key(m, mm.n);
        // probabilities are >= 0: IEEE bit order == numeric order; descending via ~
        probk[t] = ~static_cast<uint64_t>(__double_as_longlong(p < 0 ? 0.0 : p));
        idx[t] = m;
    }
}

__global__ void direct_kernel(const double* __restrict__ src, int from_amps, const uint64_t* __restrict__ fixed,
                              MemberMap mm, int64_t n_groups, uint64_t seed, uint64_t* __restrict__ out,
                              int64_t* __restrict__ bad) {
    const int64_t per = int64_t{1} << mm.l;
    for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < n_groups;
         g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double* s = src + (from_amps ? 2 : 1) * g * per;
        auto prob = [&](int64_t i) {
            if (!from_amps) return s[i];
            return __dadd_rn(__dmul_rn(s[2 * i], s[2 * i]), __dmul_rn(s[2 * i + 1], s[2 * i + 1]));
        };
        double total = 0.0;
        for (int64_t i = 0; i < per; ++i) total = __dadd_rn(total, prob(i));
        if (!(total > 0.0)) {
            atomicMin(reinterpret_cast<unsigned long long*>(bad), static_cast<unsigned long long>(g));
            out[g] = 0;
            continue;
        }
        // g-th draw of Rng(seed): counter-based SplitMix64
        uint64_t z = seed + static_cast<uint64_t>(g + 1) * 0x9e3779b97f4a7c15ull;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        z ^= z >> 31;
        double u = __dmul_rn(static_cast<double>(z >> 11) * 0x1.0p-53, total);
        int64_t pick = per - 1;
        for (int64_t i = 0; i < per; ++i) {
            u = __dsub_rn(u, prob(i));
            if (u <= 0.0) {
                pick = i;
                break;
            }
        }
        out[g] = member_index(mm, fixed[g], static_cast<uint64_t>(pick));
    }
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
    return mm;
}

struct DevBuf {
    void* p = nullptr;
    explicit DevBuf(size_t bytes) {
        if (cudaMalloc(&p, std::max<size_t>(bytes, 16)) != cudaSuccess)
            throw Failure{RCSG_ERR_DEVICE, "cudaMalloc failed in post-processing"};
    }
    ~DevBuf() { cudaFree(p); }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

}  // namespace

void topk_select(const rcsg_candidates& cs, const double* d_src, bool from_amps, uint64_t k,
                 uint64_t* out, cudaStream_t st) {
    const MemberMap mm = make_map(cs);
    const int64_t total = static_cast<int64_t>(cs.n_groups) << cs.l;
    if (k < 1 || k > static_cast<uint64_t>(total))
        throw Failure{RCSG_ERR_CONFIG, "top-k size k=" + std::to_string(k) + " outside [1, " +
                                           std::to_string(total) + "]"};
    DevBuf fixed(cs.n_groups * sizeof(uint64_t));
    CUDA_OK(cudaMemcpyAsync(fixed.p, cs.group_fixed, cs.n_groups * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
    DevBuf lex(total * 8), lex2(total * 8), pk(total * 8), pk2(total * 8), id(total * 8), id2(total * 8);
    const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
    topk_keys_kernel<<<grid, 256, 0, st>>>(d_src, from_amps, fixed.as<uint64_t>(), mm, total, lex.as<uint64_t>(),
                                           pk.as<uint64_t>(), id.as<uint64_t>());
    // pass 1: order by lexicographic key (ascending); pass 2: stable order by
    // the inverted probability bits, i.e. probability descending with ties
    // left in lexicographic order (sampling.cpp:97-100).
    size_t tmp_bytes = 0;
    CUDA_OK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, lex.as<uint64_t>(), lex2.as<uint64_t>(),
                                            pk.as<uint64_t>(), pk2.as<uint64_t>(), total, 0, cs.n_qubits, st));
    size_t tmp2 = 0;
    CUDA_OK(cub::DeviceRadixSort::SortPairs(nullptr, tmp2, pk2.as<uint64_t>(), pk.as<uint64_t>(),
                                            id.as<uint64_t>(), id2.as<uint64_t>(), total, 0, 64, st));
    DevBuf tmp(std::max(tmp_bytes, tmp2));
    // sort (lexkey, probkey) pairs and (lexkey, index) pairs with the same keys:
    // radix sort is stable and deterministic, so both produce the same order.
    CUDA_OK(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, lex.as<uint64_t>(), lex2.as<uint64_t>(),
                                            pk.as<uint64_t>(), pk2.as<uint64_t>(), total, 0, cs.n_qubits, st));
    CUDA_OK(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, lex.as<uint64_t>(), lex2.as<uint64_t>(),
                                            id.as<uint64_t>(), id2.as<uint64_t>(), total, 0, cs.n_qubits, st));
    // pass 2: stable order by prob key (= prob descending)
    CUDA_OK(cub::DeviceRadixSort::SortPairs(tmp.p, tmp2, pk2.as<uint64_t>(), pk.as<uint64_t>(),
                                            id2.as<uint64_t>(), id.as<uint64_t>(), total, 0, 64, st));
    CUDA_OK(cudaMemcpyAsync(out, id.p, k * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
}

void direct_sample(const rcsg_candidates& cs, const double* d_src, bool from_amps, uint64_t seed,
                   uint64_t* out, cudaStream_t st) {
    const MemberMap mm = make_map(cs);
    const int64_t G = static_cast<int64_t>(cs.n_groups);
    DevBuf fixed(G * sizeof(uint64_t)), d_out(G * sizeof(uint64_t)), bad(sizeof(int64_t));
    CUDA_OK(cudaMemcpyAsync(fixed.p, cs.group_fixed, G * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
    const int64_t none = LLONG_MAX;
    CUDA_OK(cudaMemcpyAsync(bad.p, &none, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    const int grid = static_cast<int>(std::min<int64_t>((G + 127) / 128, 148 * 8));
    direct_kernel<<<std::max(grid, 1), 128, 0, st>>>(d_src, from_amps, fixed.as<uint64_t>(), mm, G, seed,
                                                     d_out.as<uint64_t>(), bad.as<int64_t>());
    int64_t b = none;
    CUDA_OK(cudaMemcpyAsync(&b, bad.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaMemcpyAsync(out, d_out.p, G * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
    if (b != none)
        throw Failure{RCSG_ERR_CONFIG, "group " + std::to_string(b) + " has zero total probability; cannot sample"};
}

}  // namespace rcsg
