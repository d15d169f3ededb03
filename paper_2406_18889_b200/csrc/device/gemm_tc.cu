// tcgen05 tensor-core complex GEMM for sm_100a (kind::tf32, fp32 accumulate in TMEM).
//
//   C[v][m][n] = sum_k A[ia(v)][m][k] * B[ib(v)][n][k]      (planar complex, K-major)
//
// 4M complex product on real tensor cores: two TMEM accumulators per tile,
//   Re += Ar*Br + (-Ai)*Bi      (the second MMA sets the A-negate bit of the
//   Im += Ar*Bi +   Ai *Br       instruction descriptor)
// CTA = 128 threads: warp 0 lane 0 issues TMA (4 planes per stage into a
// 3-4 stage SWIZZLE_128B ring guarded by mbarriers), warp 1 lane 0 issues the
// MMAs and commits stages back to the producer; after the last k-block all four
// warps drain TMEM (tcgen05.ld 32x32b) and store fp32 planes with a non-finite
// check.  Small output grids use split-K with a fixed-order reduction kernel
// (deterministic).  Replaces the reference's naive ikj complex<double> loop
// (contraction_engine.cpp:115-123).
#include <cuda.h>

#include <algorithm>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>

#include "kernels.cuh"

namespace rcsg {
namespace {

constexpr int kBM = 128;
// K elements per 128-B swizzle row: 32 fp32 (tf32 path) or 64 bf16
template <typename E>
constexpr int KBK = 128 / static_cast<int>(sizeof(E));
// K elements per stage row of RB bytes (128: SWIZZLE_128B; 64 / 32: narrow-K tiles)
template <typename E, int RB>
constexpr int kbk = RB / static_cast<int>(sizeof(E));
constexpr int kThreads = 128;

// SM count of the current device (cached per device: one process may drive several GPUs)
int num_sms() {
    static std::atomic<int> cache[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    int n = cache[dev].load(std::memory_order_relaxed);
    if (!n) {
        n = 148;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        cache[dev].store(n, std::memory_order_relaxed);
    }
    return n;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// The same wait with a suspend-time hint: the thread sleeps in the barrier
// until the phase completes (or ~20 us pass) instead of re-issuing try_wait,
// which frees issue slots for the other epilogue warps of the SM sub-partition.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(20000)
        : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

// K-major SWIZZLE_128B shared-memory matrix descriptor (tcgen05 "version 1"):
// start address >> 4, SBO = 1024 B between 8-row atoms, layout type 2.
// K-major operand tile with RB-byte rows, swizzled to match the TMA box:
// SBO = one 8-row core-matrix group; layout type 2 / 4 / 6 = SWIZZLE_128B / 64B / 32B
template <int RB = 128>
__device__ __forceinline__ uint64_t smem_desc(const void* p) {
    const uint64_t addr = smem_u32(p);
    uint64_t d = (addr >> 4) & 0x3FFF;
    d |= uint64_t{1} << 16;                            // LBO (unused for swizzled K-major)
    d |= uint64_t{(8 * RB) >> 4} << 32;                // SBO
    d |= uint64_t{1} << 46;                            // descriptor version (sm_100)
    d |= uint64_t{RB == 128 ? 2u : (RB == 64 ? 4u : 6u)} << 61;
    return d;
}

// Instruction descriptor: D=f32, A=B=tf32, both K-major, M=128, N=bn.
__host__ __device__ constexpr uint32_t idesc_tf32(int bn, bool neg_a) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (neg_a ? (1u << 13) : 0u) |
           (static_cast<uint32_t>(bn >> 3) << 17) | (static_cast<uint32_t>(kBM >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

// element traits: operand format code of the instruction descriptor, TMA type, MMA kind
template <typename E>
struct TcElem;
template <>
struct TcElem<float> {
    static constexpr uint32_t fmt = 2;  // TF32 (kind::tf32)
    static constexpr CUtensorMapDataType tma = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
};
template <>
struct TcElem<bf16> {
    static constexpr uint32_t fmt = 1;  // BF16 (kind::f16)
    static constexpr CUtensorMapDataType tma = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
};
template <>
struct TcElem<f16> {
    static constexpr uint32_t fmt = 0;  // F16 (kind::f16)
    static constexpr CUtensorMapDataType tma = CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
};
template <typename E>
__host__ __device__ constexpr uint32_t idesc_of(int bn, bool neg_a, int bm = kBM) {
    return (1u << 4) | (TcElem<E>::fmt << 7) | (TcElem<E>::fmt << 10) | (neg_a ? (1u << 13) : 0u) |
           (static_cast<uint32_t>(bn >> 3) << 17) | (static_cast<uint32_t>(bm >> 4) << 24);
}
// one 128 x BN x 32-byte-K MMA (8 tf32 or 16 bf16 along K)
template <typename E>
__device__ __forceinline__ void mma_e(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    if constexpr (sizeof(E) == 4) mma_tf32(tmem_d, da, db, idesc, acc);
    else mma_bf16(tmem_d, da, db, idesc, acc);
}

// CTA pair (cta_group::2): the leader CTA issues one 256 x N MMA over both
// CTAs' shared memory (A: 128 rows in each CTA, B: N/2 rows in each); each
// CTA's TMEM receives its own 128 accumulator rows
template <typename E>
__device__ __forceinline__ void mma_pair(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    if constexpr (sizeof(E) == 4)
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "setp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n"
            "}\n" ::"r"(tmem_d),
            "l"(da), "l"(db), "r"(idesc), "r"(acc));
    else
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "setp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
            "}\n" ::"r"(tmem_d),
            "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

// arrive on the same barrier in both CTAs of the pair once the issued MMAs complete
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(static_cast<uint16_t>(3))
        : "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// shared::cluster address of this CTA's shared variable `p` in CTA `rank`
__device__ __forceinline__ uint32_t cluster_addr(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}

__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_bar) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}

// TMA load whose completion is signalled on the pair leader's barrier
// (`bar` is a shared::cluster address, possibly in the peer CTA)
__device__ __forceinline__ void tma_load_3d_pair(void* dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                                                 int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
        "%3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

struct TcParams {
    int64_t m, n, k;        // per-variant GEMM shape
    int64_t batch;          // C variants
    int64_t mt, nt;         // tiles per variant
    int m_fast;             // raster order: m-tile index varies fastest
    int64_t k_chunk;        // k elements per split
    int splits;
    const int32_t* ia;      // gather tables (mode 2) or nullptr
    const int32_t* ib;
    int a_batched, b_batched;
    void* c;                // C re-plane (element type) or split-K workspace (float)
    int64_t c_plane, c_batch;
    int64_t ws_split;       // workspace elements per split (split-K), 0 otherwise
    int32_t step;
    int32_t* fault;
    OutMap om;              // output scatter map (applied when not split)
    int32_t scale_exp;      // outputs stored times 2^scale_exp (fp16 mode)
    int32_t round_tf32;     // tf32 mode: outputs rounded to tf32 (tf32_rn)
    int32_t b_resident;     // B identical for every tile: loaded once per stage slot
    int32_t ng;             // persistent kernel: epilogue warp groups (tiles in flight), 1 / 2 / 4
    int32_t group;          // grouped raster: G "hi" tiles per super-row (0: plain mixed-radix order)
    const int32_t* vperm;   // batched GEMMs with a shared operand: variant order (nullptr: none); the
                            // raster then runs over m-tiles x (variant, n-tile) so that the tiles in
                            // flight read the same shared-operand panels (see coord_at)
    int32_t tm;             // persistent kernel: rows per tile (128, or 256 for a CTA pair)
    int32_t blk_planes;     // TMA-store map per C plane (map_c: Re, map_c2: Im; offsets within a plane)
    int32_t blk;            // 4-byte outputs stored by TMA from shared memory in 16 x 16 blocks: 1 =
                            // columns 0-3 at output bits 0-3 (64-B column runs), 2 = rows 0-3 at bits 0-3
    int32_t seg;            // > 0: k-blocks per TMEM accumulation segment; the epilogue sums the
                            // segments in fp32 registers (split tf32: short tensor-core accumulation chains)
    int32_t sleepy;         // persistent kernel: producer / MMA threads wait with a suspend-time hint
                            // (they stop competing for issue slots with the epilogue warps)
    int32_t epi;            // staged epilogue (2-byte E): 0 off, 1 column runs, 2 column runs
                            // with row-fast lanes, 3 row runs (see store_chunk_staged)
};

// Store one 32-column chunk of one plane (0 Re, 1 Im) of a thread's row: to the
// split-K workspace (fp32, row-major), or to C (element type) row-major
// (vectorised for fp32) or through the output scatter map into the
// consumer's layout.
template <typename E, int CW = 32>
__device__ __forceinline__ bool store_chunk(const TcParams& p, int split, int64_t v, int64_t row, int64_t col0,
                                            float* x, int plane, const int64_t* tn_lo, int64_t row_off,
                                            int64_t col_base) {
    bool bad = false;
    if (p.ws_split) {  // raw partials; the reduction scales and checks
#pragma unroll
        for (int i = 0; i < CW; ++i) bad |= !isfinite(x[i]);
        float* pr = static_cast<float*>(p.c) + split * p.ws_split + v * p.c_batch + plane * p.c_plane + row * p.n + col0;
        for (int i = 0; i < CW && col0 + i < p.n; ++i) pr[i] = x[i];
        return bad;
    }
    if (p.scale_exp) {
        const float sc = exp2f(static_cast<float>(p.scale_exp));
#pragma unroll
        for (int i = 0; i < CW; ++i) x[i] *= sc;
    }
    if (p.round_tf32) {
#pragma unroll
        for (int i = 0; i < CW; ++i) x[i] = tf32_rn(x[i]);
    }
#pragma unroll
    for (int i = 0; i < CW; ++i) bad |= unstorable<E>(x[i]);
    E* cpl = static_cast<E*>(p.c) + v * p.c_batch + plane * p.c_plane;
    if (!p.om.scatter) {
        E* pr = cpl + row * p.n + col0;
        if constexpr (sizeof(E) == 4) {
            if (col0 + CW <= p.n && (p.n & 3) == 0) {
#pragma unroll
                for (int i = 0; i < CW; i += 4)
                    *reinterpret_cast<float4*>(pr + i) = make_float4(x[i], x[i + 1], x[i + 2], x[i + 3]);
                return bad;
            }
        }
        for (int i = 0; i < CW && col0 + i < p.n; ++i) store_c(pr + i, x[i]);
        return bad;
    }
    const int64_t base = row_off + col_base;
    const int sh = p.om.n_pos[0];
    const bool contig = p.om.n_bits >= 5 && p.om.n_pos[1] == sh + 1 && p.om.n_pos[2] == sh + 2 &&
                        p.om.n_pos[3] == sh + 3 && p.om.n_pos[4] == sh + 4;
    if (col0 + CW <= p.n && contig) {
        // column bits contiguous at bit sh (sh == 0: per-thread contiguous run)
#pragma unroll
        for (int i = 0; i < CW; ++i) store_c(cpl + base + (static_cast<int64_t>(i) << sh), x[i]);
    } else {
        for (int i = 0; i < CW && col0 + i < p.n; ++i) store_c(cpl + base + tn_lo[i], x[i]);
    }
    return bad;
}

// Staged epilogue for 2-byte outputs.  A lane holds one row's 32 columns;
// when the output's fastest bits are column bits (epi 1, 2) or row bits
// (epi 3) the scalar stores hit one 32-B sector per 2-B element.  Instead the
// warp parks its 32x32 chunk in shared memory and re-reads it as 16-B vectors
// of 8 output-contiguous elements: 8 consecutive columns of one row (epi 1:
// lanes sweep a row's 4 vectors, epi 2: lanes sweep 32 rows, for outputs whose
// row bit 0 sits right above a 3-bit column run) or 8 consecutive rows of one
// column (epi 3).
constexpr int kEpiPitch = 32;  // elements per staged row (64 B)
constexpr int kEpiWarpElems = 32 * kEpiPitch;
// staged element (r, c): 16-B slot c/8 XOR-swizzled by bits 1-2 and 3-4 of r,
// so row writes, row-vector reads and 8-row column gathers (epi 3) are all
// bank-conflict-free
__device__ __forceinline__ int epi_at(int r, int c) {
    return r * kEpiPitch + ((((c >> 3) ^ (r >> 1) ^ (r >> 3)) & 3) << 3) + (c & 7);
}

template <typename E>
__device__ __forceinline__ uint4 pack8(const float* x) {
    union {
        E e[8];
        uint4 u;
    } t;
#pragma unroll
    for (int i = 0; i < 8; ++i) store_c(&t.e[i], x[i]);
    return t.u;
}

// one plane of a warp's 32x32 chunk (rows row0.., columns col0..)
template <typename E, int CW = 32>
__device__ __forceinline__ bool store_chunk_staged(const TcParams& p, int64_t v, int64_t row0, E* stage, float* x,
                                                   int plane, const int64_t* tn_lo, int lane, int64_t my_off,
                                                   int64_t col_base) {
    bool bad = false;
    if (p.scale_exp) {
        const float sc = exp2f(static_cast<float>(p.scale_exp));
#pragma unroll
        for (int i = 0; i < CW; ++i) x[i] *= sc;
    }
    const bool live = row0 + lane < p.m;
    if (live) {  // one range check on the max magnitude, plus NaN
        float mx = 0.f;
        bool nan = false;
#pragma unroll
        for (int i = 0; i < CW; ++i) {
            mx = fmaxf(mx, fabsf(x[i]));
            nan |= x[i] != x[i];
        }
        bad = nan || unstorable<E>(mx);
    }
    E* const base = static_cast<E*>(p.c) + v * p.c_batch + plane * p.c_plane + col_base;
    // the chunk is 32 rows x CW columns = 4 * CW / 8 sixteen-byte vectors per lane... per warp:
    // NIT rounds of 32 lanes; VPR vectors per row
    constexpr int VPR = CW / 8, NIT = CW / 8;
#pragma unroll
    for (int i = 0; i < VPR; ++i)
        *reinterpret_cast<uint4*>(stage + epi_at(lane, 8 * i)) = pack8<E>(x + 8 * i);
    __syncwarp();
    if (p.epi == 3) {
        // 8 consecutive rows of a column pair (c, c + 1): eight 32-bit reads give
        // both columns' vectors (low / high halves), half the shared loads of a
        // per-column 16-bit gather
#pragma unroll
        for (int it = 0; it < NIT / 2; ++it) {
            const int id = it * 32 + lane;
            const int c = (id >> 2) * 2, r = (id & 3) * 8;
            uint32_t w[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) w[e] = *reinterpret_cast<const uint32_t*>(stage + epi_at(r + e, c));
            uint4 v0, v1;
            v0.x = __byte_perm(w[0], w[1], 0x5410), v1.x = __byte_perm(w[0], w[1], 0x7632);
            v0.y = __byte_perm(w[2], w[3], 0x5410), v1.y = __byte_perm(w[2], w[3], 0x7632);
            v0.z = __byte_perm(w[4], w[5], 0x5410), v1.z = __byte_perm(w[4], w[5], 0x7632);
            v0.w = __byte_perm(w[6], w[7], 0x5410), v1.w = __byte_perm(w[6], w[7], 0x7632);
            const int64_t roff = __shfl_sync(0xffffffffu, my_off, r);
            if (row0 + r < p.m) {
                *reinterpret_cast<uint4*>(base + roff + tn_lo[c]) = v0;
                *reinterpret_cast<uint4*>(base + roff + tn_lo[c + 1]) = v1;
            }
        }
        __syncwarp();
        return bad;
    }
#pragma unroll
    for (int it = 0; it < NIT; ++it) {  // 8 consecutive columns of row r
        const int id = it * 32 + lane;
        const int cv = p.epi == 2 ? (id >> 5) : (id % VPR);
        const int r = p.epi == 2 ? (id & 31) : (id / VPR);
        const uint4 val = *reinterpret_cast<const uint4*>(stage + epi_at(r, cv * 8));
        const int64_t roff = __shfl_sync(0xffffffffu, my_off, r);
        if (row0 + r < p.m) *reinterpret_cast<uint4*>(base + roff + tn_lo[cv * 8]) = val;
    }
    __syncwarp();
    return bad;
}

// Staged epilogue for 4-byte (fp32 / tf32-mode) outputs, the same idea with a
// 32-row x 16-column fp32 half-chunk per warp (64-B rows, 16-B slots, the
// 2-byte layout's swizzle): epi 1 = column runs of >= 4 at output bit 0
// (lanes write 16-B vectors along rows), epi 3 = row runs of >= 4 (lanes
// gather 4 rows of one column into a 16-B vector).
constexpr int kEpiPitch4 = 16;  // floats per staged row (64 B)
constexpr int kEpiWarpElems4 = 32 * kEpiPitch4;
__device__ __forceinline__ int epi_at4(int r, int c) {
    return r * kEpiPitch4 + ((((c >> 2) ^ (r >> 1) ^ (r >> 3)) & 3) << 2) + (c & 3);
}

template <int CW = 32>
__device__ __forceinline__ bool store_chunk_staged4(const TcParams& p, int64_t v, int64_t row0, float* stage,
                                                    float* x, int plane, const int64_t* tn_lo, int lane,
                                                    int64_t my_off, int64_t col_base) {
    bool bad = false;
    if (p.scale_exp) {
        const float sc = exp2f(static_cast<float>(p.scale_exp));
#pragma unroll
        for (int i = 0; i < CW; ++i) x[i] *= sc;
    }
    if (p.round_tf32) {
        // non-finite check by FFMA (x * 0 is NaN exactly for Inf / NaN x) before and after an
        // integer round-to-nearest-away to tf32 (cvt.rna.tf32.f32 is emulated with a per-element
        // Inf test; the checks here cover NaN inputs and a rounding overflow instead)
        float z0 = 0.f, z1 = 0.f;
#pragma unroll
        for (int i = 0; i < CW; ++i) {
            z0 = fmaf(x[i], 0.f, z0);
            x[i] = __uint_as_float((__float_as_uint(x[i]) + 0x1000u) & 0xffffe000u);
            z1 = fmaf(x[i], 0.f, z1);
        }
        if (row0 + lane < p.m) bad = z0 != z0 || z1 != z1;
    } else if (row0 + lane < p.m) {
#pragma unroll
        for (int i = 0; i < CW; ++i) bad |= !isfinite(x[i]);
    }
    float* const base = static_cast<float*>(p.c) + v * p.c_batch + plane * p.c_plane + col_base;
#pragma unroll
    for (int h = 0; h < CW / 16; ++h) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
            *reinterpret_cast<float4*>(stage + epi_at4(lane, 4 * i)) =
                make_float4(x[16 * h + 4 * i], x[16 * h + 4 * i + 1], x[16 * h + 4 * i + 2], x[16 * h + 4 * i + 3]);
        __syncwarp();
        if (p.epi == 3) {
#pragma unroll
            for (int it = 0; it < 4; ++it) {  // 4 consecutive rows of one column
                const int id = it * 32 + lane;
                const int c = id >> 3, r = (id & 7) * 4;
                float4 val;
                val.x = stage[epi_at4(r, c)];
                val.y = stage[epi_at4(r + 1, c)];
                val.z = stage[epi_at4(r + 2, c)];
                val.w = stage[epi_at4(r + 3, c)];
                const int64_t roff = __shfl_sync(0xffffffffu, my_off, r);
                if (row0 + r < p.m) *reinterpret_cast<float4*>(base + roff + tn_lo[16 * h + c]) = val;
            }
        } else {
#pragma unroll
            for (int it = 0; it < 4; ++it) {  // 4 consecutive columns of one row
                const int id = it * 32 + lane;
                const int cv = id & 3, r = id >> 2;
                const float4 val = *reinterpret_cast<const float4*>(stage + epi_at4(r, 4 * cv));
                const int64_t roff = __shfl_sync(0xffffffffu, my_off, r);
                if (row0 + r < p.m) *reinterpret_cast<float4*>(base + roff + tn_lo[16 * h + 4 * cv]) = val;
            }
        }
        __syncwarp();
    }
    return bad;
}

// TMA-store epilogue for 4-byte outputs with a 64-B run at output bits 0-3 (p.blk
// 1: four column bits, 2: four row bits): the warp stages each 16-column half of
// its 32 x CW chunk as two 16 x 16 blocks (SWIZZLE_64B, the run innermost) and two
// lanes issue one TMA tensor store each through map_c, a 5-D view of the C buffer
// {element offset, then one extent-2 dimension per output bit of the other four
// bits 0-3 (stride 2^pos)}.  The global writes leave the LSU / L1 path: the staged
// epilogue spends it on shared loads plus 16-B stores, and those steps were
// L1-pipe-bound (profiles/r02/ncu_s3/cfg4_k8_*).
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t smem, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(smem)
                 : "memory");
}
__device__ __forceinline__ void tma_store_5d(const CUtensorMap* map, uint32_t smem, int x) {
    asm volatile(
        "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %2, %2, %2}], [%3];" ::"l"(
            reinterpret_cast<uint64_t>(map)),
        "r"(x), "r"(0), "r"(smem)
        : "memory");
}

template <int CW = 32>
__device__ __forceinline__ bool store_chunk_tma4(const TcParams& p, const CUtensorMap* map_c, int64_t v, int64_t row0,
                                                 float* stage, float* x, int plane, const int64_t* tn_lo, int lane,
                                                 int64_t my_off, int64_t col_base) {
    if (p.scale_exp) {
        const float sc = exp2f(static_cast<float>(p.scale_exp));
#pragma unroll
        for (int i = 0; i < CW; ++i) x[i] *= sc;
    }
    bool bad = false;
    if (p.round_tf32) {
        float z0 = 0.f, z1 = 0.f;
#pragma unroll
        for (int i = 0; i < CW; ++i) {
            z0 = fmaf(x[i], 0.f, z0);
            x[i] = __uint_as_float((__float_as_uint(x[i]) + 0x1000u) & 0xffffe000u);
            z1 = fmaf(x[i], 0.f, z1);
        }
        bad = z0 != z0 || z1 != z1;
    } else {
#pragma unroll
        for (int i = 0; i < CW; ++i) bad |= !isfinite(x[i]);
    }
    const int r = lane & 15;
    float* blk = stage + (lane >> 4) * 256;  // lanes 0-15: block 0, lanes 16-31: block 1 (1 KB each)
    const bool issuer = (lane & 15) == 0;
    const int64_t base_el = (p.blk_planes ? 0 : plane * p.c_plane) + v * p.c_batch + my_off + col_base;
#pragma unroll
    for (int h = 0; h < CW / 16; ++h) {
        if (issuer) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // the buffer is free
        __syncwarp();
        if (p.blk & 1) {  // [row][16 columns]: 64-B rows, 16-B slot i ^ (row / 2) % 4
#pragma unroll
            for (int i = 0; i < 4; ++i)
                *reinterpret_cast<float4*>(blk + r * 16 + ((i ^ ((r >> 1) & 3)) << 2)) =
                    make_float4(x[16 * h + 4 * i], x[16 * h + 4 * i + 1], x[16 * h + 4 * i + 2], x[16 * h + 4 * i + 3]);
        } else {  // [column][16 rows]: lane r scatters its 16 columns into the 64-B column rows
#pragma unroll
            for (int c = 0; c < 16; ++c) blk[c * 16 + ((((r >> 2) ^ (c >> 1)) & 3) << 2) + (r & 3)] = x[16 * h + c];
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (issuer) {
            const int64_t off = base_el + tn_lo[16 * h];  // block origin (row and column bits 0-3 zero)
            if (p.blk >= 3) tma_store_2d(map_c, smem_u32(blk), 0, static_cast<int>(off >> 4));  // one 1-KB run
            else tma_store_5d(map_c, smem_u32(blk), static_cast<int>(off));
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    return bad;
}

// The same for 2-byte outputs with a 64-B (32-element) run at output bits 0-4 (p.blk
// 1: five column bits, 2: five row bits; 3 / 4: the other index's four low bits at
// 5-8, one 1-KB run per block through a 2-D map).  Column runs: two 16-row x 32-column
// blocks per chunk (lanes 0-15, 16-31); row runs: two 16-column x 32-row blocks
// (every lane writes its row into both).
template <typename E>
__device__ __forceinline__ bool store_chunk_tma2(const TcParams& p, const CUtensorMap* map_c, int64_t v,
                                                 int64_t row0, E* stage, float* x, int plane, const int64_t* tn_lo,
                                                 int lane, int64_t my_off, int64_t col_base) {
    constexpr int CW = 32;
    if (p.scale_exp) {
        const float sc = exp2f(static_cast<float>(p.scale_exp));
#pragma unroll
        for (int i = 0; i < CW; ++i) x[i] *= sc;
    }
    float mx = 0.f;
    bool nan = false;
#pragma unroll
    for (int i = 0; i < CW; ++i) {
        mx = fmaxf(mx, fabsf(x[i]));
        nan |= x[i] != x[i];
    }
    const bool bad = nan || unstorable<E>(mx);
    const int64_t base_el = (p.blk_planes ? 0 : plane * p.c_plane) + v * p.c_batch + col_base;
    if (lane == 0 || lane == 16) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // buffer free
    __syncwarp();
    if (p.blk & 1) {  // [row][32 columns] per 16-row block: 64-B rows, 16-B slot i ^ (row / 2) % 4
        const int r = lane & 15;
        E* blk = stage + (lane >> 4) * 512;
#pragma unroll
        for (int i = 0; i < 4; ++i)
            *reinterpret_cast<uint4*>(blk + r * 32 + ((i ^ ((r >> 1) & 3)) << 3)) = pack8<E>(x + 8 * i);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if ((lane & 15) == 0) {
            const int64_t off = base_el + my_off;  // block origin: row bits 0-3 and column bits 0-4 zero
            if (p.blk >= 3) tma_store_2d(map_c, smem_u32(blk), 0, static_cast<int>(off >> 5));
            else tma_store_5d(map_c, smem_u32(blk), static_cast<int>(off));
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    } else {  // [column][32 rows] per 16-column block: lane = row, slot (row / 8) ^ (column / 2) % 4
#pragma unroll
        for (int c = 0; c < CW; ++c) {
            E* blk = stage + (c >> 4) * 512;
            const int cc = c & 15;
            store_c(blk + cc * 32 + ((((lane >> 3) ^ (cc >> 1)) & 3) << 3) + (lane & 7), x[c]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        const int64_t roff = __shfl_sync(0xffffffffu, my_off, 0);
        if (lane == 0 || lane == 16) {
            const int b = lane >> 4;
            const int64_t off = base_el + roff + tn_lo[16 * b];  // row bits 0-4 and column bits 0-3 zero
            E* blk = stage + b * 512;
            if (p.blk >= 3) tma_store_2d(map_c, smem_u32(blk), 0, static_cast<int>(off >> 5));
            else tma_store_5d(map_c, smem_u32(blk), static_cast<int>(off));
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    return bad;
}

template <int BN, int STAGES, int RB = 128, int NPL = 2, int CG = 1>
struct Smem {
    static constexpr int kATile = kBM * RB;  // bytes per A plane tile (RB-byte rows)
    static constexpr int kBTile = (BN / CG) * RB;  // a CTA pair holds half of B's N rows in each CTA
    // NPL planes per operand: {Ar, Ai, Br, Bi} (4M), {Ar, Ai, Ar+Ai, Br, Bi, Br+Bi} (3M)
    static constexpr int kStage = NPL * kATile + NPL * kBTile;
    static constexpr int kBytes = STAGES * kStage + 1024 /*align*/ + 512 /*barriers*/;
    // persistent kernel: + staged-epilogue buffers of the 8 epilogue warps (2-byte E)
    template <typename E>
    static constexpr int kPBytes = kBytes + (sizeof(E) == 2 ? 16 * kEpiWarpElems * 2 : 16 * kEpiWarpElems4 * 4);
};

template <int BN, int STAGES, typename E>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap map_ar, const __grid_constant__ CUtensorMap map_ai,
                   const __grid_constant__ CUtensorMap map_br, const __grid_constant__ CUtensorMap map_bi,
                   const TcParams p) {
    using S = Smem<BN, STAGES>;
    extern __shared__ uint8_t smem_raw[];
    // offset the __shared__ array itself (not via an integer cast) so the compiler keeps
    // the shared address space and emits LDS/STS rather than generic loads and stores
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * S::kStage);
    uint64_t* empty = full + STAGES;
    uint64_t* done = empty + STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __shared__ int64_t tn_lo[32];
    if (threadIdx.x < 32) tn_lo[threadIdx.x] = out_col_off(p.om, threadIdx.x);
    // tile coordinates
    // raster: the tile dimension with fewer tiles varies fastest, so CTAs that
    // run together share the larger operand's tile through L2
    int64_t t = blockIdx.x;
    const int split = static_cast<int>(t % p.splits);
    t /= p.splits;
    int64_t ntile, mtile;
    if (p.m_fast) {
        mtile = t % p.mt;
        t /= p.mt;
        ntile = t % p.nt;
        t /= p.nt;
    } else {
        ntile = t % p.nt;
        t /= p.nt;
        mtile = t % p.mt;
        t /= p.mt;
    }
    const int64_t v = t;
    const int m0 = static_cast<int>(mtile * kBM), n0 = static_cast<int>(ntile * BN);
    const int av = p.ia ? p.ia[v] : (p.a_batched ? static_cast<int>(v) : 0);
    const int bv = p.ib ? p.ib[v] : (p.b_batched ? static_cast<int>(v) : 0);
    const int64_t k_begin = split * p.k_chunk;
    const int64_t k_end = min(p.k, k_begin + p.k_chunk);
    const int kblocks = static_cast<int>((k_end - k_begin + KBK<E> - 1) / KBK<E>);

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(2 * BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    pdl_enter();  // the prologue above touched no global memory

    if (warp == 0 && lane == 0) {
        // ---- TMA producer
        for (int kb = 0; kb < kblocks; ++kb) {
            const int s = kb % STAGES;
            const uint32_t round = kb / STAGES;
            if (kb >= STAGES) mbar_wait(&empty[s], (round - 1) & 1);
            uint8_t* st = smem + s * S::kStage;
            mbar_expect_tx(&full[s], S::kStage);
            const int kc = static_cast<int>(k_begin) + kb * KBK<E>;
            tma_load_3d(st, &map_ar, &full[s], kc, m0, av);
            tma_load_3d(st + S::kATile, &map_ai, &full[s], kc, m0, av);
            tma_load_3d(st + 2 * S::kATile, &map_br, &full[s], kc, n0, bv);
            tma_load_3d(st + 2 * S::kATile + S::kBTile, &map_bi, &full[s], kc, n0, bv);
        }
    } else if (warp == 1 && lane == 0) {
        // ---- MMA issuer (single thread)
        constexpr uint32_t id_pos = idesc_of<E>(BN, false), id_neg = idesc_of<E>(BN, true);
        const uint32_t t_re = tmem, t_im = tmem + BN;
        for (int kb = 0; kb < kblocks; ++kb) {
            const int s = kb % STAGES;
            mbar_wait(&full[s], (kb / STAGES) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint8_t* st = smem + s * S::kStage;
            const uint64_t dar = smem_desc(st), dai = smem_desc(st + S::kATile);
            const uint64_t dbr = smem_desc(st + 2 * S::kATile), dbi = smem_desc(st + 2 * S::kATile + S::kBTile);
#pragma unroll
            for (int j = 0; j < 4; ++j) {  // 4 x 32 B along K per 128-B row
                const uint64_t o = static_cast<uint64_t>(j * 32) >> 4;  // 8 tf32 = 32 B along K
                const uint32_t acc = (kb > 0 || j > 0) ? 1u : 0u;
                mma_e<E>(t_re, dar + o, dbr + o, id_pos, acc);
                mma_e<E>(t_re, dai + o, dbi + o, id_neg, 1u);
                mma_e<E>(t_im, dar + o, dbi + o, id_pos, acc);
                mma_e<E>(t_im, dai + o, dbr + o, id_pos, 1u);
            }
            mma_commit(&empty[s]);  // frees the stage once these MMAs retire
        }
        mma_commit(done);
    }
    __syncwarp();

    // ---- epilogue: all 4 warps, warp w owns TMEM lanes [32w, 32w+32) = tile rows
    mbar_wait(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int64_t row = m0 + warp * 32 + lane;
    bool bad = false;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
        float re[32], im[32];
        const uint32_t lane_base = static_cast<uint32_t>(warp * 32) << 16;
        tmem_ld32(tmem + lane_base + c0, re);
        tmem_ld32(tmem + lane_base + BN + c0, im);
        if (kblocks == 0) {
#pragma unroll
            for (int i = 0; i < 32; ++i) re[i] = im[i] = 0.f;
        }
        if (row < p.m) {
            const int64_t ro = out_row_off(p.om, p.n, row), cb = out_col_off(p.om, n0 + c0);
            bad |= store_chunk<E>(p, split, v, row, n0 + c0, re, 0, tn_lo, ro, cb);
            bad |= store_chunk<E>(p, split, v, row, n0 + c0, im, 1, tn_lo, ro, cb);
        }
    }
    if (bad && p.fault && p.splits == 1) atomicMin(p.fault, p.step);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN));
}

// ---- persistent variant: one CTA per SM loops over tiles; the accumulators are
// double-buffered in TMEM (2 x {Re, Im} x BN columns) so the four epilogue
// warps drain tile i while the MMA warp already accumulates tile i+1.
//   warp 0: TMA producer   warp 1: MMA issuer   warps 2-5: epilogue (TMEM lane quarter = warp % 4)
constexpr int kPThreads = 576;  // 2 role warps + 16 epilogue warps (4 per TMEM lane quarter: plane x half)

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// OR of a 64-bit value across the warp
__device__ __forceinline__ int64_t warp_or64(int64_t v) {
    const uint32_t lo = __reduce_or_sync(0xffffffffu, static_cast<uint32_t>(v));
    const uint32_t hi = __reduce_or_sync(0xffffffffu, static_cast<uint32_t>(static_cast<uint64_t>(v) >> 32));
    return static_cast<int64_t>((static_cast<uint64_t>(hi) << 32) | lo);
}
// scatter of bits [lo_bit, bits) of a warp-uniform x: lane j places bit j
__device__ __forceinline__ int64_t warp_scatter(const int8_t* pos, int bits, int lo_bit, int64_t x, int lane) {
    int64_t c = 0;
    if (lane >= lo_bit && lane < bits) c = ((x >> lane) & int64_t{1}) << pos[lane];
    return warp_or64(c);
}

struct TileCoord {
    int64_t v;
    int m0, n0, split, kblocks;
    int64_t k_begin;
};

template <int BN, typename E, int RB = 128>
__device__ __forceinline__ TileCoord tile_coord(const TcParams& p, int64_t t64) {
    // tile counts fit 32 bits (the host checks): 32-bit div/mod, not the 64-bit routine
    TileCoord c;
    uint32_t t = static_cast<uint32_t>(t64);
    const uint32_t splits = static_cast<uint32_t>(p.splits), mt = static_cast<uint32_t>(p.mt),
                   nt = static_cast<uint32_t>(p.nt);
    uint32_t q = splits == 1 ? t : t / splits;
    c.split = static_cast<int>(t - q * splits);
    t = q;
    uint32_t ntile, mtile;
    if (p.m_fast) {
        q = t / mt;
        mtile = t - q * mt;
        t = q;
        q = t / nt;
        ntile = t - q * nt;
        t = q;
    } else {
        q = t / nt;
        ntile = t - q * nt;
        t = q;
        q = t / mt;
        mtile = t - q * mt;
        t = q;
    }
    c.v = t;
    c.m0 = static_cast<int>(mtile * p.tm);
    c.n0 = static_cast<int>(ntile * BN);
    c.k_begin = c.split * p.k_chunk;
    const int64_t k_end = min(p.k, c.k_begin + p.k_chunk);
    c.kblocks = static_cast<int>((k_end - c.k_begin + kbk<E, RB> - 1) / kbk<E, RB>);
    return c;
}

// Tile index t = ((split * n_v + v) * n_hi + hi) * n_lo + lo, with (lo, hi) =
// (m tile, n tile) when m_fast else (n tile, m tile).  A CTA walks t = blockIdx.x,
// blockIdx.x + gridDim.x, ...: the digits advance by gridDim.x's mixed-radix
// digits with carries, so no division per tile.
struct TileIter {
    uint32_t split, lo, hi, v;           // current digits
    uint32_t d_split, d_lo, d_hi, d_v;   // gridDim.x in the same radix
    uint32_t splits, n_lo, n_hi, n_v;
    __device__ void init(const TcParams& p, uint32_t t, uint32_t step) {
        splits = static_cast<uint32_t>(p.splits);
        n_lo = static_cast<uint32_t>(p.m_fast ? p.mt : p.nt);
        n_hi = static_cast<uint32_t>(p.m_fast ? p.nt : p.mt);
        n_v = static_cast<uint32_t>(p.batch < 1 ? 1 : p.batch);
        if (p.vperm) {  // lo = (variant, n-tile) in vperm order, hi = m-tiles
            n_lo = static_cast<uint32_t>(p.nt) * n_v;
            n_hi = static_cast<uint32_t>(p.mt);
            n_v = 1;
        }
        // split is the slowest digit: the tiles in flight together work on the
        // same K range, so their A / B panels are shared through L2
        auto digits = [&](uint32_t x, uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
            b = x % n_lo;
            x /= n_lo;
            c = x % n_hi;
            x /= n_hi;
            d = x % n_v;
            a = x / n_v;
        };
        digits(t, split, lo, hi, v);
        digits(step, d_split, d_lo, d_hi, d_v);
    }
    __device__ __forceinline__ void next() {
        lo += d_lo;
        uint32_t c = lo >= n_lo;
        lo -= c ? n_lo : 0;
        hi += d_hi + c;
        c = hi >= n_hi;
        hi -= c ? n_hi : 0;
        v += d_v + c;
        c = v >= n_v;
        v -= c ? n_v : 0;
        split += d_split + c;
    }
    // Grouped raster (long-K GEMMs): consecutive tiles - the ones in flight
    // together - cover G "hi" tiles x (in flight / G) "lo" tiles instead of a few
    // whole "lo" rows, so each operand panel streamed from HBM is shared by ~G
    // (resp. in flight / G) CTAs through L2.  One 32-bit division chain per
    // tile, for tiles that run >= 32 k-blocks.
    template <int BN, typename E, int RB>
    __device__ __forceinline__ TileCoord coord_at(const TcParams& p, int64_t t64) const {
        if (!p.group) return coord<BN, E, RB>(p);
        TileCoord c;
        const uint32_t t = static_cast<uint32_t>(t64);
        const uint32_t per_v = n_lo * n_hi, per_split = per_v * n_v;
        c.split = static_cast<int>(t / per_split);
        const uint32_t q = t - static_cast<uint32_t>(c.split) * per_split;
        const uint32_t v = q / per_v, r = q - v * per_v;
        const uint32_t G = static_cast<uint32_t>(p.group);
        const uint32_t grp = r / (G * n_lo), rg = r - grp * (G * n_lo);
        const uint32_t first = grp * G, gsz = min(G, n_hi - first);
        const uint32_t hi_d = first + rg % gsz, lo_d = rg / gsz;
        if (p.vperm) {  // G m-tiles x (in flight / G) consecutive variants of the sorted order
            const uint32_t nt = static_cast<uint32_t>(p.nt), j = lo_d / nt;
            c.v = static_cast<uint32_t>(__ldg(p.vperm + j));
            c.m0 = static_cast<int>(hi_d * p.tm);
            c.n0 = static_cast<int>((lo_d - j * nt) * BN);
        } else {
            const uint32_t mtile = p.m_fast ? lo_d : hi_d, ntile = p.m_fast ? hi_d : lo_d;
            c.v = v;
            c.m0 = static_cast<int>(mtile * p.tm);
            c.n0 = static_cast<int>(ntile * BN);
        }
        c.k_begin = c.split * p.k_chunk;
        const int64_t k_end = min(p.k, c.k_begin + p.k_chunk);
        c.kblocks = static_cast<int>((k_end - c.k_begin + kbk<E, RB> - 1) / kbk<E, RB>);
        return c;
    }
    template <int BN, typename E, int RB>
    __device__ __forceinline__ TileCoord coord(const TcParams& p) const {
        TileCoord c;
        c.split = static_cast<int>(split);
        const uint32_t mtile = p.m_fast ? lo : hi, ntile = p.m_fast ? hi : lo;
        c.v = v;
        c.m0 = static_cast<int>(mtile * p.tm);
        c.n0 = static_cast<int>(ntile * BN);
        c.k_begin = c.split * p.k_chunk;
        const int64_t k_end = min(p.k, c.k_begin + p.k_chunk);
        c.kblocks = static_cast<int>((k_end - c.k_begin + kbk<E, RB> - 1) / kbk<E, RB>);
        return c;
    }
};

// THREE (3M complex product): T1 = Ar Br, T2 = Ai Bi, T3 = (Ar+Ai)(Br+Bi), then
// Re = T1 - T2, Im = T3 - T1 - T2 in the epilogue - three real MMAs per K slice
// instead of four, with the operand sum planes staged by the host-side pre-pass.
// VAR: 0 = 4M, 1 = 3M (three accumulators), 2 = split tf32 (3xTF32, two accumulators)
template <int VAR>
constexpr uint32_t tc_nbuf(int bn) {
    return (512 / ((VAR == 1 ? 3 : 2) * bn)) < 4 ? (512 / ((VAR == 1 ? 3 : 2) * bn)) : 4;
}
constexpr uint32_t pow2_ceil(uint32_t x) {
    uint32_t r = 32;
    while (r < x) r <<= 1;
    return r;
}

// CG = 2: CTA-pair variant (cluster of 2 on one TPC, cta_group::2).  Tiles are
// 256 x BN; each CTA loads its 128 A rows and BN/2 of the B rows, the leader
// CTA's producer expects both CTAs' bytes on its full barrier, the leader's MMA
// thread issues 256 x BN MMAs and commits to both CTAs' barriers, and each
// CTA's epilogue drains its own TMEM rows; the peer's epilogue warps release a
// TMEM buffer on the leader's tempty barrier.  Per CTA, a k-block moves half
// of B's bytes of the 1-CTA tile for the same MMA work.
// VAR = 2 (split tf32, "3xTF32"): fp32 operands x = hi + lo, hi = rna_tf32(x),
// lo = rna_tf32(x - hi), staged by a pre-pass (map_ar / map_ai / map_br / map_bi
// read the hi planes, map_as / map_as2 / map_bs / map_bs2 the lo planes); each
// real product is hi*hi + hi*lo + lo*hi (12 MMAs per K slice for the complex
// 4M form), which carries ~fp32 accuracy on the tf32 tensor cores.
template <int BN, int STAGES, typename E, int RB, int VAR = 0, int CG = 1>
__global__ void __launch_bounds__(kPThreads, 1)
    gemm_tc_persistent(const __grid_constant__ CUtensorMap map_ar, const __grid_constant__ CUtensorMap map_ai,
                       const __grid_constant__ CUtensorMap map_br, const __grid_constant__ CUtensorMap map_bi,
                       const __grid_constant__ CUtensorMap map_as, const __grid_constant__ CUtensorMap map_bs,
                       const __grid_constant__ CUtensorMap map_as2, const __grid_constant__ CUtensorMap map_bs2,
                       const __grid_constant__ CUtensorMap map_c, const __grid_constant__ CUtensorMap map_c2,
                       const TcParams p, int64_t total_tiles) {
    constexpr bool THREE = VAR == 1, SPLIT = VAR == 2;
    constexpr int NPL = VAR == 0 ? 2 : (VAR == 1 ? 3 : 4);  // shared-memory planes per operand
    constexpr int NACC = VAR == 1 ? 3 : 2;                  // TMEM accumulators per tile
    static_assert(CG == 1 || VAR == 0, "3M / split tf32 have no CTA-pair variant");
    static_assert(!SPLIT || sizeof(E) == 4, "split tf32 needs fp32 operands");
    using S = Smem<BN, STAGES, RB, NPL, CG>;
    // TMEM accumulator buffers ({Re, Im}, or {T1, T2, T3} for 3M): as many as fit in
    // 512 columns (max 4), so the MMA runs ahead of the epilogue by NBUF - 1 tiles
    constexpr uint32_t NBUF = tc_nbuf<VAR>(BN);
    constexpr uint32_t kCols = pow2_ceil(NBUF * NACC * BN);
    // epilogue groups = tiles in flight (NBUF % NG == 0), chosen by the host (p.ng: 1, 2 or 4)
    const int NG = p.ng;
    extern __shared__ uint8_t smem_raw[];
    // offset the __shared__ array itself (not via an integer cast) so the compiler keeps
    // the shared address space and emits LDS/STS rather than generic loads and stores
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * S::kStage);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + NBUF;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + NBUF);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = CG == 2 ? cluster_rank() : 0u;  // CTA pair: 0 = leader
    // tiles are walked per CTA pair (cluster): both CTAs of a pair take the same tiles
    const uint32_t unit = blockIdx.x / CG, n_units = gridDim.x / CG;
    __shared__ int64_t tn_lo[32];
    if (threadIdx.x < 32) tn_lo[threadIdx.x] = out_col_off(p.om, threadIdx.x);
    if (threadIdx.x == 32) {  // fetch the TMA descriptors while the CTA sets up
        for (const CUtensorMap* m : {&map_ar, &map_ai, &map_br, &map_bi, &map_as, &map_bs, &map_as2, &map_bs2})
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
    }

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < static_cast<int>(NBUF); ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], CG * 16 / NG);  // one epilogue group (per CTA of the pair) drains each buffer
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 0) {
        if constexpr (CG == 2) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(kCols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(kCols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if constexpr (CG == 2) cluster_sync();  // the peer's barriers are initialised before any remote signal
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    pdl_enter();  // the prologue above touched no global memory

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer
            uint32_t it = 0;
            TileIter ti;
            ti.init(p, unit, n_units);
            for (int64_t t = unit; t < total_tiles; t += n_units, ti.next()) {
                const TileCoord c = ti.coord_at<BN, E, RB>(p, t);
                const int av = p.ia ? p.ia[c.v] : (p.a_batched ? static_cast<int>(c.v) : 0);
                const int bv = p.ib ? p.ib[c.v] : (p.b_batched ? static_cast<int>(c.v) : 0);
                for (int kb = 0; kb < c.kblocks; ++kb, ++it) {
                    const int s = it % STAGES;
                    if (it >= STAGES) {
                        if (p.sleepy) mbar_wait_sleep(&empty[s], ((it / STAGES) - 1) & 1);
                        else mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
                    }
                    uint8_t* st = smem + s * S::kStage;
                    const int kc = static_cast<int>(c.k_begin) + kb * kbk<E, RB>;
                    if constexpr (CG == 2) {
                        // both CTAs' bytes complete on the leader's full barrier
                        if (rank == 0) mbar_expect_tx(&full[s], 2 * S::kStage);
                        const uint32_t bar = cluster_addr(&full[s], 0);
                        const int ma = c.m0 + static_cast<int>(rank) * kBM, nb = c.n0 + static_cast<int>(rank) * (BN / 2);
                        tma_load_3d_pair(st, &map_ar, bar, kc, ma, av);
                        tma_load_3d_pair(st + S::kATile, &map_ai, bar, kc, ma, av);
                        uint8_t* sb = st + NPL * S::kATile;
                        tma_load_3d_pair(sb, &map_br, bar, kc, nb, bv);
                        tma_load_3d_pair(sb + S::kBTile, &map_bi, bar, kc, nb, bv);
                    } else {
                        // B resident: the same single B tile for every tile (one N tile, one
                        // K block, unbatched B) is loaded once into each stage slot
                        const bool load_b = !(p.b_resident && it >= STAGES);
                        mbar_expect_tx(&full[s], load_b ? S::kStage : NPL * S::kATile);
                        tma_load_3d(st, &map_ar, &full[s], kc, c.m0, av);
                        tma_load_3d(st + S::kATile, &map_ai, &full[s], kc, c.m0, av);
                        if constexpr (THREE || SPLIT) tma_load_3d(st + 2 * S::kATile, &map_as, &full[s], kc, c.m0, av);
                        if constexpr (SPLIT) tma_load_3d(st + 3 * S::kATile, &map_as2, &full[s], kc, c.m0, av);
                        if (load_b) {
                            uint8_t* sb = st + NPL * S::kATile;
                            tma_load_3d(sb, &map_br, &full[s], kc, c.n0, bv);
                            tma_load_3d(sb + S::kBTile, &map_bi, &full[s], kc, c.n0, bv);
                            if constexpr (THREE || SPLIT) tma_load_3d(sb + 2 * S::kBTile, &map_bs, &full[s], kc, c.n0, bv);
                            if constexpr (SPLIT) tma_load_3d(sb + 3 * S::kBTile, &map_bs2, &full[s], kc, c.n0, bv);
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {  // ---- MMA issuer (the pair's leader CTA)
            constexpr uint32_t id_pos = idesc_of<E>(BN, false, kBM * CG), id_neg = idesc_of<E>(BN, true, kBM * CG);
            uint32_t it = 0, j = 0;
            TileIter ti;
            ti.init(p, unit, n_units);
            for (int64_t t = unit; t < total_tiles; t += n_units, ti.next()) {
              const TileCoord c = ti.coord_at<BN, E, RB>(p, t);
              // one TMEM buffer per segment of seg k-blocks (the whole tile unless p.seg > 0)
              const int seg = p.seg > 0 ? p.seg : (c.kblocks > 0 ? c.kblocks : 1);
              for (int s0 = 0;;) {
                const uint32_t ab = j % NBUF;
                if (j >= NBUF) {
                    if (p.sleepy) mbar_wait_sleep(&tempty[ab], ((j / NBUF) - 1) & 1);
                    else mbar_wait(&tempty[ab], ((j / NBUF) - 1) & 1);
                }
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t t_re = tmem + ab * NACC * BN, t_im = t_re + BN;  // 3M: T1, T2 (, T3 = t_re + 2 BN)
                const int s1 = min(c.kblocks, s0 + seg);
                for (int kb = s0; kb < s1; ++kb, ++it) {
                    const int s = it % STAGES;
                    if (p.sleepy) mbar_wait_sleep(&full[s], (it / STAGES) & 1);
                    else mbar_wait(&full[s], (it / STAGES) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint8_t* st = smem + s * S::kStage;
                    const uint8_t* sb = st + NPL * S::kATile;
                    const uint64_t dar = smem_desc<RB>(st), dai = smem_desc<RB>(st + S::kATile);
                    const uint64_t dbr = smem_desc<RB>(sb), dbi = smem_desc<RB>(sb + S::kBTile);
#pragma unroll
                    for (int jj = 0; jj < RB / 32; ++jj) {  // 32-B K slices (one MMA K each)
                        const uint64_t o = static_cast<uint64_t>(jj * 32) >> 4;
                        const uint32_t acc = (kb > s0 || jj > 0) ? 1u : 0u;
                        if constexpr (THREE) {
                            const uint64_t das = smem_desc<RB>(st + 2 * S::kATile), dbs = smem_desc<RB>(sb + 2 * S::kBTile);
                            mma_e<E>(t_re, dar + o, dbr + o, id_pos, acc);           // T1 = Ar Br
                            mma_e<E>(t_im, dai + o, dbi + o, id_pos, acc);           // T2 = Ai Bi
                            mma_e<E>(t_re + 2 * BN, das + o, dbs + o, id_pos, acc);  // T3 = As Bs
                        } else if constexpr (SPLIT) {
                            // lo planes: Ar_lo, Ai_lo at A tiles 2, 3; Br_lo, Bi_lo at B tiles 2, 3.
                            // Small cross terms first, then hi * hi
                            const uint64_t darl = smem_desc<RB>(st + 2 * S::kATile), dail = smem_desc<RB>(st + 3 * S::kATile);
                            const uint64_t dbrl = smem_desc<RB>(sb + 2 * S::kBTile), dbil = smem_desc<RB>(sb + 3 * S::kBTile);
                            mma_e<E>(t_re, darl + o, dbr + o, id_pos, acc);   // Re += Arl Br + Ar Brl + Ar Br
                            mma_e<E>(t_re, dar + o, dbrl + o, id_pos, 1u);
                            mma_e<E>(t_re, dail + o, dbi + o, id_neg, 1u);    //      - (Ail Bi + Ai Bil + Ai Bi)
                            mma_e<E>(t_re, dai + o, dbil + o, id_neg, 1u);
                            mma_e<E>(t_re, dar + o, dbr + o, id_pos, 1u);
                            mma_e<E>(t_re, dai + o, dbi + o, id_neg, 1u);
                            mma_e<E>(t_im, darl + o, dbi + o, id_pos, acc);   // Im += Arl Bi + Ar Bil + Ar Bi
                            mma_e<E>(t_im, dar + o, dbil + o, id_pos, 1u);
                            mma_e<E>(t_im, dail + o, dbr + o, id_pos, 1u);    //      + Ail Br + Ai Brl + Ai Br
                            mma_e<E>(t_im, dai + o, dbrl + o, id_pos, 1u);
                            mma_e<E>(t_im, dar + o, dbi + o, id_pos, 1u);
                            mma_e<E>(t_im, dai + o, dbr + o, id_pos, 1u);
                        } else if constexpr (CG == 2) {
                            mma_pair<E>(t_re, dar + o, dbr + o, id_pos, acc);
                            mma_pair<E>(t_re, dai + o, dbi + o, id_neg, 1u);
                            mma_pair<E>(t_im, dar + o, dbi + o, id_pos, acc);
                            mma_pair<E>(t_im, dai + o, dbr + o, id_pos, 1u);
                        } else {
                            mma_e<E>(t_re, dar + o, dbr + o, id_pos, acc);
                            mma_e<E>(t_re, dai + o, dbi + o, id_neg, 1u);
                            mma_e<E>(t_im, dar + o, dbi + o, id_pos, acc);
                            mma_e<E>(t_im, dai + o, dbr + o, id_pos, 1u);
                        }
                    }
                    if constexpr (CG == 2) mma_commit_pair(&empty[s]);
                    else mma_commit(&empty[s]);
                }
                if constexpr (CG == 2) mma_commit_pair(&tfull[ab]);
                else mma_commit(&tfull[ab]);
                ++j;
                s0 += seg;
                if (s0 >= c.kblocks) break;
              }
            }
        }
    } else {  // ---- epilogue warps 2..17: two groups of 8 take alternate tiles; TMEM lane quarter warp % 4
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        const int sub = (warp - 2) >> 2;  // 0..3
        // NG = 1: all 16 warps on each tile (plane x column half); NG = 2: groups of 8 warps,
        // one plane each, all columns; NG = 4: groups of 4 warps, both planes
        const int grp = NG == 4 ? sub : (NG == 2 ? (sub >> 1) : 0);
        const int plane_lo = NG == 4 ? 0 : (sub & 1), plane_hi = NG == 4 ? 2 : plane_lo + 1;
        const int col_lo = NG == 1 ? (sub >> 1) * (BN / 2) : 0, col_hi = NG == 1 ? col_lo + BN / 2 : BN;
        E* stage = reinterpret_cast<E*>(smem + S::kBytes - 1024) +
                   (warp - 2) * (sizeof(E) == 2 ? kEpiWarpElems : kEpiWarpElems4);
        // output row offset = tile part (bits >= 7 of the row, warp-uniform) + this
        // lane's part (bits 0..6, fixed), when the map's row bits cover a tile
        const int local = q * 32 + lane;
        const bool split_rows = p.om.scatter && p.om.m_bits >= 7;
        const int64_t lane_off = split_rows ? scatter_bits(p.om.m_pos, 7, local) : 0;
        bool bad = false;
        uint32_t j = 0;
        TileIter ti;
        const int64_t t0 = unit + static_cast<int64_t>(grp) * n_units;
        ti.init(p, static_cast<uint32_t>(t0), NG * n_units);
        j = static_cast<uint32_t>(grp);
        const uint32_t tempty_leader = CG == 2 ? cluster_addr(tempty, 0) : 0u;  // tempty[0] in the leader
        for (int64_t t = t0; t < total_tiles; t += NG * static_cast<int64_t>(n_units), j += NG, ti.next()) {
            TileCoord c = ti.coord_at<BN, E, RB>(p, t);
            c.m0 += static_cast<int>(rank) * kBM;  // this CTA's accumulator rows
            const uint32_t ab = j % NBUF;
            const int64_t row = c.m0 + local;
            int64_t row_off;
            if (!p.om.scatter) row_off = row * p.n;
            else if (split_rows)
                row_off = (static_cast<int64_t>(c.m0) >> p.om.m_bits) * out_row_vstride(p.om) +
                          warp_scatter(p.om.m_pos, p.om.m_bits, 7, c.m0, lane) + lane_off;
            else row_off = row < p.m ? out_row_off(p.om, p.n, row) : 0;
            mbar_wait_sleep(&tfull[ab], (j / NBUF) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            // store one CW-column chunk of one plane (x: this lane's row)
            auto store_x = [&](auto cw_tag, int plane, int c0, int64_t col_base, float* x) {
                constexpr int CW = decltype(cw_tag)::value;
                const int64_t col0 = c.n0 + c0;  // multiple of CW
                if constexpr (sizeof(E) == 2) {
                    if constexpr (CW == 32) {
                        if (p.blk && p.splits == 1 && col0 + CW <= p.n && c.m0 + q * 32 + 32 <= p.m) {
                            bad |= store_chunk_tma2<E>(p, plane && p.blk_planes ? &map_c2 : &map_c, c.v, c.m0 + q * 32, stage, x, plane, tn_lo, lane,
                                                       row_off, col_base);
                            return;
                        }
                    }
                    if (p.epi && p.splits == 1 && col0 + CW <= p.n) {
                        if (p.blk)  // the buffer may still be read by an earlier TMA store
                            if (lane == 0 || lane == 16) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                        __syncwarp();
                        bad |= store_chunk_staged<E, CW>(p, c.v, c.m0 + q * 32, stage, x, plane, tn_lo, lane,
                                                         row < p.m ? row_off : 0, col_base);
                        return;
                    }
                } else {
                    if (p.blk && p.splits == 1 && col0 + CW <= p.n && c.m0 + q * 32 + 32 <= p.m) {
                        bad |= store_chunk_tma4<CW>(p, plane && p.blk_planes ? &map_c2 : &map_c, c.v, c.m0 + q * 32, reinterpret_cast<float*>(stage), x,
                                                    plane, tn_lo, lane, row_off, col_base);
                        return;
                    }
                    if (p.epi && p.splits == 1 && col0 + CW <= p.n) {
                        if (p.blk)  // the buffer may still be read by an earlier TMA store
                            if ((lane & 15) == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                        __syncwarp();
                        bad |= store_chunk_staged4<CW>(p, c.v, c.m0 + q * 32, reinterpret_cast<float*>(stage), x,
                                                       plane, tn_lo, lane, row < p.m ? row_off : 0, col_base);
                        return;
                    }
                }
                if (row < p.m)
                    bad |= store_chunk<E, CW>(p, c.split, c.v, row, col0, x, plane, tn_lo, row_off, col_base);
            };
            auto col_base_of = [&](int64_t col0, int cw_bits) {
                // single column tile (nt == 1): the first chunk's offset is 0 for every tile (no warp reductions)
                if (p.nt == 1 && col0 == 0) return int64_t{0};
                return p.om.scatter ? warp_scatter(p.om.n_pos, p.om.n_bits, cw_bits, col0, lane) +
                                          (col0 >> p.om.n_bits) * p.om.n_vstride
                                    : col0;
            };
            if constexpr (SPLIT) {
                if (p.seg > 0) {
                    // segmented accumulation (host: NG = 1, BN <= 64): this warp's one chunk
                    // (plane, column half) summed over the tile's K segments in fp32 registers
                    constexpr int CWS = BN / 2 < 32 ? BN / 2 : 32;
                    const int plane = sub & 1, c0 = (sub >> 1) * (BN / 2);
                    const int nseg = c.kblocks > 0 ? (c.kblocks + p.seg - 1) / p.seg : 1;
                    float acc[CWS], x[16];
                    for (int sg = 0; sg < nseg; ++sg, ++j) {
                        const uint32_t abs = j % NBUF;
                        mbar_wait_sleep(&tfull[abs], (j / NBUF) & 1);
                        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                        const uint32_t addr =
                            tmem + (static_cast<uint32_t>(q * 32) << 16) + abs * NACC * BN + plane * BN + c0;
#pragma unroll
                        for (int h = 0; h < CWS / 16; ++h) {  // 16 columns at a time (registers)
                            tmem_ld16(addr + 16 * h, x);
#pragma unroll
                            for (int i = 0; i < 16; ++i) acc[16 * h + i] = sg ? acc[16 * h + i] + x[i] : x[i];
                        }
                        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&tempty[abs]);
                    }
                    if (c.n0 + c0 < p.n)
                        store_x(std::integral_constant<int, CWS>{}, plane, c0, col_base_of(c.n0 + c0, CWS == 32 ? 5 : 4),
                                acc);
                    j -= NG;  // the loop header advances j by NG per tile
                    continue;
                }
            }
            mbar_wait_sleep(&tfull[ab], (j / NBUF) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            // one chunk = CW columns of one plane; BN = 32 tiles drained by a group of
            // warps that owns all columns (NG >= 2) take the whole 32-column row at once
            auto chunk = [&](auto cw_tag, int plane, int c0, int64_t col_base) {
                constexpr int CW = decltype(cw_tag)::value;
                const uint32_t lanes = tmem + (static_cast<uint32_t>(q * 32) << 16) + ab * NACC * BN + c0;
                float x[CW];
                auto ld = [&](uint32_t addr, float* v) {
                    if constexpr (CW == 32) tmem_ld32(addr, v);
                    else tmem_ld16(addr, v);
                };
                if constexpr (THREE) {  // Re = T1 - T2, Im = T3 - T1 - T2
                    float y[CW];
                    ld(lanes + (plane == 0 ? 0 : 2 * BN), x);
                    ld(lanes + (plane == 0 ? BN : 0), y);
#pragma unroll
                    for (int i = 0; i < CW; ++i) x[i] -= y[i];
                    if (plane == 1) {
                        ld(lanes + BN, y);
#pragma unroll
                        for (int i = 0; i < CW; ++i) x[i] -= y[i];
                    }
                } else {
                    ld(lanes + plane * BN, x);
                }
                store_x(cw_tag, plane, c0, col_base, x);
            };
            if (BN == 32 && NG != 1 && p.n >= 32) {
#pragma unroll 1
                for (int plane = plane_lo; plane < plane_hi; ++plane)
                    chunk(std::integral_constant<int, 32>{}, plane, 0, col_base_of(c.n0, 5));
            } else {
                constexpr int CWD = BN / 2 < 32 ? BN / 2 : 32;  // 16 when BN = 32 and NG = 1
#pragma unroll 1
                for (int plane = plane_lo; plane < plane_hi; ++plane)
#pragma unroll 1
                    for (int c0 = col_lo; c0 < col_hi && c.n0 + c0 < p.n; c0 += CWD)  // no chunks past n
                        chunk(std::integral_constant<int, CWD>{}, plane, c0, col_base_of(c.n0 + c0, CWD == 32 ? 5 : 4));
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                if constexpr (CG == 2) mbar_arrive_cluster(tempty_leader + ab * 8u);
                else mbar_arrive(&tempty[ab]);
            }
        }
        if (bad && p.fault && p.splits == 1) atomicMin(p.fault, p.step);
        if (p.blk && (lane & 15) == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // TMA stores done
    }
    __syncwarp();
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if constexpr (CG == 2) {
        cluster_sync();  // neither CTA frees TMEM or exits while the pair still signals it
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols));
    } else {
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols));
    }
}

// ---- host side
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess || !f)
            throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
        return reinterpret_cast<EncodeFn>(f);
    }();
    return fn;
}

// 3D map over a [batch][rows][k] plane, box {RB bytes of k, box_rows, 1}, swizzled to RB.
template <typename E, int RB = 128>
CUtensorMap make_map(const void* base, int64_t k, int64_t rows, int64_t batch, int box_rows) {
    CUtensorMap m;
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(rows),
                          static_cast<cuuint64_t>(std::max<int64_t>(batch, 1))};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(k * sizeof(E)), static_cast<cuuint64_t>(k * rows * sizeof(E))};
    cuuint32_t box[3] = {static_cast<cuuint32_t>(kbk<E, RB>), static_cast<cuuint32_t>(box_rows), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = encode_fn()(&m, TcElem<E>::tma, 3, const_cast<void*>(base), dims, strides,
                                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   RB == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                             : (RB == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B),
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return m;
}

// Staged-epilogue kind for a 2-byte output layout (see store_chunk_staged).
int epilogue_kind(const OutMap& om, int64_t n) {
    if (n % 32) return 0;
    int cr = 0, rr = 0;  // column / row bits at output bits 0, 1, 2, ...
    if (!om.scatter) {
        cr = 64;
    } else {
        while (cr < om.n_bits && om.n_pos[cr] == cr) ++cr;
        while (rr < om.m_bits && om.m_pos[rr] == rr) ++rr;
    }
    if (cr >= 3) return (cr == 3 && om.scatter && om.m_bits > 0 && om.m_pos[0] == 3) ? 2 : 1;
    if (rr >= 3) return 3;
    return 0;
}

// Staged-epilogue kind for a 4-byte output layout (see store_chunk_staged4):
// 16-B vectors need runs of >= 4 column (epi 1) or row (epi 3) bits at bit 0.
int epilogue_kind4(const OutMap& om, int64_t n) {
    if (n % 16) return 0;
    int cr = 0, rr = 0;
    if (!om.scatter) {
        cr = 64;
    } else {
        while (cr < om.n_bits && om.n_pos[cr] == cr) ++cr;
        while (rr < om.m_bits && om.m_pos[rr] == rr) ++rr;
    }
    if (cr >= 2) return 1;
    if (rr >= 2) return 3;
    return 0;
}

template <int BN, int STAGES, typename E, int RB = 128, int VAR = 0, int CG = 1>
void launch(const GemmArgs& g, cudaStream_t st, const void* a_sum = nullptr, const void* b_sum = nullptr,
            const void* a_sum2 = nullptr, const void* b_sum2 = nullptr) {
    constexpr bool THREE = VAR == 1;
    using S = Smem<BN, STAGES, RB, VAR == 0 ? 2 : (VAR == 1 ? 3 : 4), CG>;
    const int64_t a_rows = g.ia ? g.m : g.m;  // rows per A variant (mode 1 folds variants into m)
    const int64_t a_batches = g.a_batch ? std::max<int64_t>(1, g.a_plane / std::max<int64_t>(g.a_batch, 1)) : 1;
    const int64_t b_batches = g.b_batch ? std::max<int64_t>(1, g.b_plane / std::max<int64_t>(g.b_batch, 1)) : 1;
    const E* a = static_cast<const E*>(g.a);
    const E* b = static_cast<const E*>(g.b);
    const CUtensorMap ar = make_map<E, RB>(a, g.k, a_rows, a_batches, kBM);
    const CUtensorMap ai = make_map<E, RB>(a + g.a_plane, g.k, a_rows, a_batches, kBM);
    const CUtensorMap br = make_map<E, RB>(b, g.k, g.n, b_batches, BN / CG);
    const CUtensorMap bi = make_map<E, RB>(b + g.b_plane, g.k, g.n, b_batches, BN / CG);
    // 3M: the Re+Im sum planes; split tf32: the lo planes (Re, Im)
    const CUtensorMap as = VAR ? make_map<E, RB>(static_cast<const E*>(a_sum), g.k, a_rows, a_batches, kBM) : ar;
    const CUtensorMap bs = VAR ? make_map<E, RB>(static_cast<const E*>(b_sum), g.k, g.n, b_batches, BN) : br;
    const CUtensorMap as2 = VAR == 2 ? make_map<E, RB>(static_cast<const E*>(a_sum2), g.k, a_rows, a_batches, kBM) : ar;
    const CUtensorMap bs2 = VAR == 2 ? make_map<E, RB>(static_cast<const E*>(b_sum2), g.k, g.n, b_batches, BN) : br;
    TcParams p{};
    p.m = g.m;
    p.n = g.n;
    p.k = g.k;
    p.batch = g.batch;
    p.tm = kBM * CG;
    p.mt = (g.m + p.tm - 1) / p.tm;
    p.nt = (g.n + BN - 1) / BN;
    p.m_fast = p.mt < p.nt ? 1 : 0;
    p.ia = g.ia;
    p.ib = g.ib;
    p.a_batched = g.a_batch != 0;
    p.b_batched = g.b_batch != 0;
    p.step = g.step;
    p.fault = g.fault;
    p.om = g.om;
    p.scale_exp = g.scale_exp;
    p.round_tf32 = g.round_tf32;
    p.epi = sizeof(E) == 2 ? epilogue_kind(g.om, g.n) : epilogue_kind4(g.om, g.n);
    if (const char* e = getenv("RCSG_TC_NO_STAGE")) if (atoi(e)) p.epi = 0;
    p.sleepy = getenv("RCSG_TC_SLEEPY") ? atoi(getenv("RCSG_TC_SLEEPY")) : 0;
    if (getenv("RCSG_DUMP_EPI")) {  // diagnostics: the output layout of every tcgen05 GEMM
        fprintf(stderr, "[rcsg-epi] m=%lld n=%lld k=%lld batch=%lld elem=%d epi=%d scatter=%d m_pos:",
                (long long)g.m, (long long)g.n, (long long)g.k, (long long)g.batch, (int)sizeof(E), p.epi,
                g.om.scatter);
        for (int j = 0; j < g.om.m_bits; ++j) fprintf(stderr, " %d", g.om.m_pos[j]);
        fprintf(stderr, " n_pos:");
        for (int j = 0; j < g.om.n_bits; ++j) fprintf(stderr, " %d", g.om.n_pos[j]);
        fprintf(stderr, "\n");
    }
    const int64_t tiles = p.mt * p.nt * g.batch;
    const int64_t kblocks = (g.k + kbk<E, RB> - 1) / kbk<E, RB>;
    // split K until the grid covers the machine (>= ~2 waves of 148 SMs), keeping >= 8 k-blocks per split;
    // then, for long-K work, keep doubling while it cuts the last-wave idle time by > 5% (wave
    // quantisation: 256 tiles on 148 SMs leave 13% of the machine idle at any split in {1, 2})
    int splits = 1;
    while (tiles * splits < 296 && kblocks / (splits * 2) >= 8) splits *= 2;
    {
        const int64_t sms = num_sms();
        auto eff = [&](int64_t units) {
            return static_cast<double>(units) / static_cast<double>(((units + sms - 1) / sms) * sms);
        };
        while (kblocks / (splits * 2) >= 64 && eff(tiles * splits * 2) > eff(tiles * splits) + 0.05) splits *= 2;
    }
    // at most max_kb k-blocks per split (RCSG_TC_MAX_KB; experiments on the accumulation chain length)
    if (const char* e = getenv("RCSG_TC_MAX_KB")) {
        const int64_t max_kb = std::max<int64_t>(1, atoll(e));
        while ((kblocks + splits - 1) / splits > max_kb && splits < 4096) splits *= 2;
    }
    const int64_t chunk_blocks = (kblocks + splits - 1) / splits;
    splits = static_cast<int>((kblocks + chunk_blocks - 1) / chunk_blocks);  // no empty split
    p.splits = splits;
    p.k_chunk = chunk_blocks * kbk<E, RB>;
    const int64_t c_elems = g.batch * g.m * g.n;  // per plane
    {
        // NBUF must be a multiple of the group count.
        constexpr int nbuf = static_cast<int>(tc_nbuf<VAR>(BN));
        // BN >= 64: all 16 epilogue warps on each tile (NG = 1) measured 5-12 % faster on the
        // HBM-bound (small-K) steps than two groups, and the same on long K; BN = 32: 4 groups
        // (profiles/r02/ng_probe)
        static const int ng_wide = getenv("RCSG_TC_NG_WIDE") ? atoi(getenv("RCSG_TC_NG_WIDE")) : 1;
        int ng = (BN == 32 && nbuf >= 4) ? 4 : ng_wide;
        if (const char* e = getenv("RCSG_TC_NG")) ng = atoi(e);
        if (ng != 1 && ng != 2 && ng != 4) ng = 1;
        while (ng > 1 && nbuf % ng) ng /= 2;
        if (VAR == 2) {
            // split tf32: TMEM accumulation segments of 16 k-blocks (K = 256), summed by the
            // epilogue in fp32 (the tensor cores' fp32 accumulation over long K chains costs
            // ~3e-9 per k-block, profiles/r02/split_acc.log); needs NG = 1 and BN <= 64
            static const int seg = getenv("RCSG_TC_SPLIT_SEG") ? atoi(getenv("RCSG_TC_SPLIT_SEG")) : 16;
            p.seg = BN <= 64 ? seg : 0;
            if (p.seg > 0) ng = 1;
        }
        p.ng = ng;
    }
    // TMA-store epilogue (store_chunk_tma4 / tma2): a 64-B run at output bits 0.. (4-byte: four
    // column (blk 1) or row (blk 2) bits; 2-byte: five), short-K GEMMs; RCSG_TC_BLK=0 disables
    CUtensorMap mc = ar, mc2 = ar;
    p.blk_planes = 0;
    {
        static const bool blk_on = !(getenv("RCSG_TC_BLK") && atoi(getenv("RCSG_TC_BLK")) == 0);
        // 2-byte outputs: opt-in (RCSG_TC_BLK2=1); measured +1 % on cfg2 fp16 and -1 to -3 % on cfg4
        // fp16 (profiles/r02/blk/ab_blk2.log), where the staged 16-B stores were not L1-bound
        const bool blk2_on = getenv("RCSG_TC_BLK2") && atoi(getenv("RCSG_TC_BLK2")) == 1;
        constexpr int RUN = sizeof(E) == 4 ? 4 : 5;  // run bits: 64 B
        constexpr int OTH = 4;                       // the other index's bits per block
        const int cw = BN / 2 < 32 ? BN / 2 : 32;    // epilogue chunk width (NG = 1)
        int kind = 0;
        // short K only (<= 16 k-blocks per tile): on long-K, compute-bound tiles the stores compete with
        // the operand loads for the TMA unit (cfg2 step 149: 5 % slower, profiles/r02/blk/ab_blk.log)
        if (blk_on && VAR == 0 && splits == 1 && chunk_blocks <= 16 && g.om.scatter &&
            (reinterpret_cast<uintptr_t>(g.c) & 255) == 0 && (sizeof(E) == 4 || (cw == 32 && p.ng == 1 && blk2_on))) {
            bool cols = g.om.n_bits >= RUN && g.om.m_bits >= OTH, rows = g.om.m_bits >= RUN && g.om.n_bits >= OTH;
            for (int j = 0; j < RUN; ++j) {
                cols = cols && g.om.n_pos[j] == j;
                rows = rows && g.om.m_pos[j] == j;
            }
            kind = cols ? 1 : (rows ? 2 : 0);
        }
        if (kind) {
            const int8_t* other = kind == 1 ? g.om.m_pos : g.om.n_pos;  // the four low bits of the other index
            bool run = true;  // at RUN..RUN+3: each block is one 1-KB run (2-D map)
            for (int j = 0; j < OTH; ++j) run &= other[j] == RUN + j;
            // coordinates are int32: the 2-D map counts 64-B rows, the 5-D one elements
            if (run && g.c_plane % (1 << RUN) == 0 && (2 * g.c_plane >> RUN) < (int64_t{1} << 31)) {
                cuuint64_t dims[2] = {cuuint64_t{1} << RUN, static_cast<cuuint64_t>(2 * g.c_plane >> RUN)};
                cuuint64_t strides[1] = {64};
                cuuint32_t box[2] = {1u << RUN, 16};
                cuuint32_t estr[2] = {1, 1};
                const CUresult r = encode_fn()(&mc, TcElem<E>::tma, 2, g.c, dims, strides, box, estr,
                                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                                               CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                kind = r == CUDA_SUCCESS ? kind + 2 : 0;
            } else if (2 * g.c_plane >= (int64_t{1} << 31)) {
                // element offsets past int32: one 5-D map per plane (RCSG_TC_BLK_PLANES=0 disables;
                // cfg4 amplitudes bit-identical, +0.9 % per slice, profiles/r02/blk/ab_planes.log)
                static const bool planes_on = !(getenv("RCSG_TC_BLK_PLANES") && atoi(getenv("RCSG_TC_BLK_PLANES")) == 0);
                bool ok = planes_on && g.c_plane < (int64_t{1} << 31) && (g.c_plane * sizeof(E)) % 256 == 0;
                for (int pl = 0; ok && pl < 2; ++pl) {
                    cuuint64_t dims[5] = {static_cast<cuuint64_t>(g.c_plane), 2, 2, 2, 2};
                    cuuint64_t strides[4];
                    for (int j = 0; j < 4; ++j) strides[j] = cuuint64_t{sizeof(E)} << other[j];
                    cuuint32_t box[5] = {1u << RUN, 2, 2, 2, 2};
                    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
                    const CUresult r = encode_fn()(pl ? &mc2 : &mc, TcElem<E>::tma, 5,
                                                   static_cast<E*>(g.c) + pl * g.c_plane, dims, strides, box, estr,
                                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                                                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                    ok = r == CUDA_SUCCESS;
                }
                if (ok) p.blk_planes = 1;
                else kind = 0;
            } else {
                cuuint64_t dims[5] = {static_cast<cuuint64_t>(2 * g.c_plane), 2, 2, 2, 2};
                cuuint64_t strides[4];
                for (int j = 0; j < 4; ++j) strides[j] = cuuint64_t{sizeof(E)} << other[j];
                cuuint32_t box[5] = {1u << RUN, 2, 2, 2, 2};
                cuuint32_t estr[5] = {1, 1, 1, 1, 1};
                const CUresult r = encode_fn()(&mc, TcElem<E>::tma, 5, g.c, dims, strides, box, estr,
                                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                                               CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                if (r != CUDA_SUCCESS) kind = 0;
            }
        }
        p.blk = kind;
    }
    {
        // grouped raster for long-K GEMMs with enough tiles in both directions
        // (RCSG_TC_GROUP: override; 0 disables)
        const int64_t n_lo = p.m_fast ? p.mt : p.nt, n_hi = p.m_fast ? p.nt : p.mt;
        int grp = (chunk_blocks >= 32 && n_lo >= 16 && n_hi >= 8) ? 8 : 0;
        // tf32 CTA pairs with a short "lo" side (15 row pairs: cfg2 step 149 unswapped): 16 "hi" tiles
        // in flight cut the DRAM reads (profiles/r02/raster_probe.log); the swapped form (29 column
        // tiles) is faster with the default 8 (profiles/r02/ab_pgroup.log)
        static const bool pair_group = !(getenv("RCSG_TC_PAIR_GROUP") && atoi(getenv("RCSG_TC_PAIR_GROUP")) == 0);
        if (pair_group && CG == 2 && sizeof(E) == 4 && chunk_blocks >= 32 && n_lo >= 8 && n_lo < 16 && n_hi >= 32)
            grp = 16;
        if (const char* e = getenv("RCSG_TC_GROUP")) grp = atoi(e);
        p.group = grp > 0 && n_hi > grp ? grp : 0;
        if (g.vperm && g.batch > 1) {  // shared-operand batch: G = 16 m-tiles x the variants in flight
            p.vperm = g.vperm;
            p.group = static_cast<int32_t>(std::min<int64_t>(16, p.mt));
        }
    }
    p.b_resident = (CG == 1 && p.nt == 1 && splits == 1 && kblocks == 1 && !g.ib && !g.b_batch &&
                    !(getenv("RCSG_TC_NO_BRES") != nullptr)) ? 1 : 0;
    if (splits == 1) {
        p.c = g.c;
        p.c_plane = g.c_plane;
        p.c_batch = g.c_batch ? g.c_batch : g.m * g.n;
        p.ws_split = 0;
    } else {
        float* ws = static_cast<float*>(device_workspace(static_cast<size_t>(splits) * 2 * c_elems * sizeof(float), st));
        p.c = ws;
        p.c_plane = c_elems;
        p.c_batch = g.m * g.n;
        p.ws_split = 2 * c_elems;
    }
    // the persistent kernel (one CTA per SM, TMEM accumulators multi-buffered so
    // the epilogue overlaps the next tile's MMAs) for every shape: on long K it
    // measured ~1.9x the one-CTA-per-tile kernel (RCSG_TC_MODE=2 selects that one)
    static const int mode = getenv("RCSG_TC_MODE") ? atoi(getenv("RCSG_TC_MODE")) : 0;
    const bool persistent = VAR != 0 || CG == 2 || mode != 2 || RB != 128;  // narrow-K, 3M, split, pairs: persistent only
    if (persistent) {
        static std::atomic<uint64_t> pconf{0};
        if (first_on_device(pconf))
            cudaFuncSetAttribute(gemm_tc_persistent<BN, STAGES, E, RB, VAR, CG>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, S::template kPBytes<E>);
        const int64_t total = tiles * splits;
        if (total >= (int64_t{1} << 31)) throw std::runtime_error("GEMM tile count exceeds 2^31");
        // one CTA (pair) per SM (pair of SMs); a pair's two CTAs walk the same tiles
        const int grid = CG * static_cast<int>(std::min<int64_t>(total, num_sms() / CG));
        if constexpr (CG == 2) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(grid);
            cfg.blockDim = dim3(kPThreads);
            cfg.dynamicSmemBytes = S::template kPBytes<E>;
            cfg.stream = st;
            cudaLaunchAttribute attr[2];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            attr[1].id = cudaLaunchAttributeClusterDimension;
            attr[1].val.clusterDim.x = 2;
            attr[1].val.clusterDim.y = 1;
            attr[1].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 2;
            cudaLaunchKernelEx(&cfg, gemm_tc_persistent<BN, STAGES, E, RB, VAR, CG>, ar, ai, br, bi, as, bs, as2, bs2,
                               mc, mc2, p, total);
        } else {
            launch_pdl(gemm_tc_persistent<BN, STAGES, E, RB, VAR>, dim3(grid), dim3(kPThreads),
                       S::template kPBytes<E>, st, ar, ai, br, bi, as, bs, as2, bs2, mc, mc2, p, total);
        }
    } else {
        static std::atomic<uint64_t> configured{0};  // function attributes are per device
        if (first_on_device(configured))
            cudaFuncSetAttribute(gemm_tc_kernel<BN, STAGES, E>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 Smem<BN, STAGES>::kBytes);
        launch_pdl(gemm_tc_kernel<BN, STAGES, E>, dim3(static_cast<unsigned>(tiles * splits)), dim3(kThreads),
                   Smem<BN, STAGES>::kBytes, st, ar, ai, br, bi, p);
    }
    if (splits > 1) launch_splitk_reduce<E>(static_cast<const float*>(p.c), p.ws_split, splits, g, st);
}

}  // namespace

bool gemm_tc_supported(const GemmArgs& g) {
    // tensor-core tiles need >= 64 rows, >= 16 columns and a 16-B aligned K stride;
    // tiny contractions stay on the SIMT kernel (launch-bound either way).
    if (g.m < 64 || g.n < 8 || g.k < 4) return false;  // narrow N: the TMA box zero-fills past n
    if (g.m * g.n * g.k * std::max<int64_t>(g.batch, 1) < (int64_t{1} << 21)) return false;
    if (g.batch > 1 && !g.ia) return false;  // batched GEMMs are always gathered here
    if (g.k > (int64_t{1} << 31) || g.m * std::max<int64_t>(g.batch, 1) > (int64_t{1} << 31)) return false;
    return true;
}

// Narrow K uses 32-B / 64-B stage rows (fewer zero-filled K columns, deeper
// stage rings) and n <= 32 the BN = 32 tiles, for every element type;
// RCSG_TC_NARROW_K=0 / RCSG_TC_NARROW_N=0 disable them
// Re + Im of a plane pair, into `out` (3M operand sum planes), 16-B vectors
template <typename E>
__global__ void plane_sum_kernel(const E* __restrict__ re, const E* __restrict__ im, E* __restrict__ out, int64_t n) {
    pdl_enter();
    constexpr int V = 16 / static_cast<int>(sizeof(E));
    const int64_t nv = n / V;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nv; i += stride) {
        const uint4 a = reinterpret_cast<const uint4*>(re)[i], b = reinterpret_cast<const uint4*>(im)[i];
        uint4 o;
        const E* pa = reinterpret_cast<const E*>(&a);
        const E* pb = reinterpret_cast<const E*>(&b);
        E* po = reinterpret_cast<E*>(&o);
#pragma unroll
        for (int j = 0; j < V; ++j) store_c(po + j, load_c(pa + j) + load_c(pb + j));
        reinterpret_cast<uint4*>(out)[i] = o;
    }
    for (int64_t i = nv * V + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
        store_c(out + i, load_c(re + i) + load_c(im + i));
}

// 3M for large unbatched GEMMs (opt-in, RCSG_TC_3M=1): the sum planes cost one
// extra pass over each operand and the MMAs drop by a quarter, but each stage
// streams six operand planes for three MMAs instead of four for four, so the
// kernel turns L2/HBM-bound: measured 1.2-2x SLOWER than 4M on every long-K
// shape of the plans (profiles/r02/gemm_3m.log).  Kept for kernels that share
// operand tiles across CTAs (multicast / 2-CTA), where the ratio flips.
template <typename E>
bool launch_3m(const GemmArgs& g, cudaStream_t st) {
    const char* env = getenv("RCSG_TC_3M");
    const bool on = env && atoi(env) != 0;
    const double flops = 8.0 * static_cast<double>(g.m) * g.n * g.k;
    if (!on || g.batch > 1 || g.ia || g.ib || g.k < 512 || g.n < 64 || flops < 2.7e11) return false;
    const int64_t a_el = g.a_plane, b_el = g.b_plane;
    const int64_t a_pad = (a_el + 127) / 128 * 128;  // keep the B sum plane 256-B aligned
    E* sums = static_cast<E*>(device_workspace(static_cast<size_t>(a_pad + b_el) * sizeof(E), st, 1));
    E* as = sums;
    E* bs = sums + a_pad;
    const E* a = static_cast<const E*>(g.a);
    const E* b = static_cast<const E*>(g.b);
    auto grid_of = [](int64_t n) {
        return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n / (16 / sizeof(E)) + 255) / 256, 148 * 8)));
    };
    launch_pdl(plane_sum_kernel<E>, dim3(grid_of(a_el)), dim3(256), 0, st, a, a + g.a_plane, as, a_el);
    launch_pdl(plane_sum_kernel<E>, dim3(grid_of(b_el)), dim3(256), 0, st, b, b + g.b_plane, bs, b_el);
    if (g.n >= 128) {  // 2 stages of 6 x 16 KB (RB = 128) measured best of the 3M tilings
        launch<128, 2, E, 128, 1>(g, st, as, bs);
    } else {
        launch<64, 5, E, 64, 1>(g, st, as, bs);
    }
    return true;
}

// CTA-pair tiles (cta_group::2, 256 x BN) for long-K GEMMs.  Measured
// (profiles/r02/gemm_pair.log, fraction of the dense peak, 1-CTA -> pair):
//   fp16 8192x8192x131072 0.71 -> 0.82 (256x256), 2048x2048x524288 0.51 -> 0.87,
//        3604x16384x4096 0.87 -> 0.93; 8192x1024x131072 stays 1-CTA (0.88)
//   tf32 the same long-K shapes 0.71 -> 0.79 and 0.43 -> 0.64 (256x256),
//        3604x16384x4096 0.93 -> 0.95 and 8192x1024x131072 0.91 -> 0.97 (256x128;
//        256x256 tiles, one TMEM buffer, lose on the shorter K)
// RCSG_TC_PAIR: unset = this policy, 0 off, 1 = 256 x 128 tiles, 2 = 256 x 256.
template <typename E>
int pair_policy(const GemmArgs& g) {
    const int64_t kb = (g.k + kbk<E, 128> - 1) / kbk<E, 128>;
    static const int64_t min_kb = getenv("RCSG_TC_PAIR_MINKB") ? atoll(getenv("RCSG_TC_PAIR_MINKB")) : 32;
    // tf32 from n = 128 (cfg4's batched 8192 x 128 x 32768 step: +1.3 % per slice, amplitudes
    // bit-identical to 1-CTA tiles, profiles/r02/ab_minn.log)
    const int64_t min_n = getenv("RCSG_TC_PAIR_MINN") ? atoll(getenv("RCSG_TC_PAIR_MINN")) : (sizeof(E) == 4 ? 128 : 256);
    if (g.m < 512 || g.n < min_n || kb < min_kb || g.k * static_cast<int64_t>(sizeof(E)) < 512) return 0;
    if (const char* e = getenv("RCSG_TC_PAIR")) return atoi(e);
    if (sizeof(E) == 2) return g.n >= 2048 ? 2 : 0;
    return (kb >= 1024 && g.n >= 2048) ? 2 : 1;
}

// C = A B^T computed as (B A^T)^T: the operands trade places and the output map's
// row and column parts swap (the 4M complex product is symmetric in A and B).
GemmArgs swapped(const GemmArgs& g) {
    GemmArgs h = g;
    h.a = g.b;
    h.b = g.a;
    h.a_plane = g.b_plane;
    h.b_plane = g.a_plane;
    h.a_batch = g.b_batch;
    h.b_batch = g.a_batch;
    h.m = g.n;
    h.n = g.m;
    OutMap& o = h.om;
    o.m_bits = g.om.n_bits;
    o.n_bits = g.om.m_bits;
    for (int j = 0; j < kMaxRank; ++j) {
        o.m_pos[j] = g.om.n_pos[j];
        o.n_pos[j] = g.om.m_pos[j];
    }
    o.n_vstride = out_row_vstride(g.om);
    o.m_vstride = g.om.n_vstride ? g.om.n_vstride : 1;  // 1: the columns never exceed 2^n_bits (unused)
    return h;
}

// A CTA-pair tile spans 256 rows: when m pads badly to 256 (cfg2 step 149: 3604 rows ->
// 3840, 6.5 % zero rows) and n is a multiple of 256, the swapped GEMM pads m to the
// column tile instead (3712 with 128-wide tiles).  Scatter outputs, unbatched only.
template <typename E>
bool swap_for_pair(const GemmArgs& g, int bn) {
    static const bool on = !(getenv("RCSG_TC_SWAP") && atoi(getenv("RCSG_TC_SWAP")) == 0);
    if (!on || !g.om.scatter || g.batch > 1 || g.ia || g.ib || g.vperm || g.n % 256 || g.m < 256) return false;
    if (g.om.n_vstride == 0 && g.n > (int64_t{1} << g.om.n_bits)) return false;
    auto waste = [](int64_t x, int64_t t) { return static_cast<double>((x + t - 1) / t * t) / static_cast<double>(x) - 1.0; };
    return waste(g.m, 256) > waste(g.m, bn) + 0.02;
}

template <typename E>
bool launch_pair(const GemmArgs& g, cudaStream_t st) {
    int mode = pair_policy<E>(g);
    if (mode != 0 && swap_for_pair<E>(g, mode == 2 ? 256 : 128)) {
        const GemmArgs h = swapped(g);
        if (pair_policy<E>(h) == mode) {
            if (mode == 2) launch<256, 3, E, 128, 0, 2>(h, st);
            else launch<128, 4, E, 128, 0, 2>(h, st);
            return true;
        }
    }
    if (mode == 0) return false;
    if (mode == 2) launch<256, 3, E, 128, 0, 2>(g, st);
    else launch<128, 4, E, 128, 0, 2>(g, st);
    return true;
}

// hi = rna_tf32(x), lo = rna_tf32(x - hi): the "big + small" split of an fp32
// operand into two tf32 values (|lo| <= 2^-11 |x|, dropped lo * lo <= 2^-22), 16-B vectors
__global__ void tf32_split_kernel(const float* __restrict__ x, float* __restrict__ hi, float* __restrict__ lo,
                                  int64_t n) {
    pdl_enter();
    const int64_t nv = n / 4;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    auto split = [](float v, float& h, float& l) {
        h = tf32_rn(v);
        l = tf32_rn(v - h);
    };
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nv; i += stride) {
        const float4 v = reinterpret_cast<const float4*>(x)[i];
        float4 h, l;
        split(v.x, h.x, l.x);
        split(v.y, h.y, l.y);
        split(v.z, h.z, l.z);
        split(v.w, h.w, l.w);
        reinterpret_cast<float4*>(hi)[i] = h;
        reinterpret_cast<float4*>(lo)[i] = l;
    }
    for (int64_t i = nv * 4 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
        split(x[i], hi[i], lo[i]);
}

// Split tf32 ("3xTF32", precision mode 3xtf32): a pre-pass writes the hi and lo
// planes of both operands (whole operand buffers in the same [Re][Im] plane
// layout, so batched / gathered variants keep their offsets), then the
// persistent kernel runs hi*hi + hi*lo + lo*hi (12 MMAs per K slice) on 64-B K rows.
void launch_split(const GemmArgs& g, cudaStream_t st) {
    const int64_t a_el = 2 * g.a_plane, b_el = 2 * g.b_plane;  // Re and Im planes
    const int64_t a_pad = (a_el + 63) / 64 * 64, b_pad = (b_el + 63) / 64 * 64;  // 256-B aligned planes
    float* ws = static_cast<float*>(
        device_workspace(static_cast<size_t>(2 * a_pad + 2 * b_pad) * sizeof(float), st, 1));
    float *ah = ws, *al = ws + a_pad, *bh = ws + 2 * a_pad, *bl = ws + 2 * a_pad + b_pad;
    auto grid_of = [](int64_t n) {
        return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n / 4 + 255) / 256, 148 * 8)));
    };
    launch_pdl(tf32_split_kernel, dim3(grid_of(a_el)), dim3(256), 0, st, static_cast<const float*>(g.a), ah, al, a_el);
    launch_pdl(tf32_split_kernel, dim3(grid_of(b_el)), dim3(256), 0, st, static_cast<const float*>(g.b), bh, bl, b_el);
    GemmArgs h = g;  // the kernel reads the hi planes as its A / B
    h.a = ah;
    h.b = bh;
    // 64-column tiles: one 32-column chunk per epilogue warp, summed over the K segments
    if (g.n > 32) launch<64, 4, float, 64, 2>(h, st, al, bl, al + g.a_plane, bl + g.b_plane);
    else launch<32, 4, float, 64, 2>(h, st, al, bl, al + g.a_plane, bl + g.b_plane);
}

template <typename E>
void launch_typed(const GemmArgs& g, cudaStream_t st) {
    if constexpr (sizeof(E) == 4) {
        if (g.split_tf32) {
            launch_split(g, st);
            return;
        }
    }
    if (launch_3m<E>(g, st)) return;
    if (launch_pair<E>(g, st)) return;
    static const bool narrow = getenv("RCSG_TC_NARROW_K") == nullptr || atoi(getenv("RCSG_TC_NARROW_K")) != 0;
    static const bool narrow_n = getenv("RCSG_TC_NARROW_N") == nullptr || atoi(getenv("RCSG_TC_NARROW_N")) != 0;
    const int64_t kb = g.k * static_cast<int64_t>(sizeof(E));  // bytes of K per row
    if (narrow_n && g.n <= 32) {  // BN = 32: every epilogue warp owns a 16-column chunk
        if (narrow && kb <= 32) launch<32, 12, E, 32>(g, st);
        else if (narrow && kb <= 64) launch<32, 8, E, 64>(g, st);
        else launch<32, 4, E>(g, st);
        return;
    }
    if (narrow && kb <= 32) {
        if (g.n >= 128) launch<128, 12, E, 32>(g, st);
        else launch<64, 12, E, 32>(g, st);
    } else if (narrow && kb <= 64) {
        if (g.n >= 128) launch<128, 6, E, 64>(g, st);
        else launch<64, 8, E, 64>(g, st);
    } else if (g.n >= 128) {
        launch<128, 3, E>(g, st);
    } else {
        launch<64, 4, E>(g, st);
    }
}

void launch_gemm_tc(const GemmArgs& g, int elem, cudaStream_t st) {
    if (elem == 1) launch_typed<bf16>(g, st);
    else if (elem == 2) launch_typed<f16>(g, st);
    else launch_typed<float>(g, st);
}

}  // namespace rcsg
