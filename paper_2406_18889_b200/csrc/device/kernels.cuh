// Device kernels of the contraction path (declarations + launch wrappers).
//
// Storage: every tensor is PLANAR complex — a real plane of N elements followed
// by an imaginary plane of N elements — with a leading "variant" axis
// (distinct group projections, see executor.cpp) outermost:
//   re[v * payload + i], im[(total) + v * payload + i].
// Storage type: double (f64), float (f32 / tf32 / 3xtf32) or bf16 (bf16).
#pragma once
#include <atomic>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>
#include <utility>

namespace rcsg {

constexpr int kMaxRank = 40;
constexpr int kMaxLeafRank = 8;

// Storage type S of the tensors vs arithmetic type Acc<S>::T: bf16 storage is
// computed and accumulated in fp32; float and double compute in themselves.
using bf16 = __nv_bfloat16;
template <typename S>
struct Acc {
    using T = S;
};
template <>
struct Acc<bf16> {
    using T = float;
};
using f16 = __half;
template <>
struct Acc<f16> {
    using T = float;
};
__device__ __forceinline__ float load_c(const float* p) { return *p; }
__device__ __forceinline__ double load_c(const double* p) { return *p; }
__device__ __forceinline__ float load_c(const bf16* p) { return __bfloat162float(*p); }
__device__ __forceinline__ void store_c(float* p, float v) { *p = v; }
__device__ __forceinline__ void store_c(double* p, double v) { *p = v; }
__device__ __forceinline__ void store_c(bf16* p, float v) { *p = __float2bfloat16_rn(v); }
__device__ __forceinline__ float load_c(const f16* p) { return __half2float(*p); }
__device__ __forceinline__ void store_c(f16* p, float v) { *p = __float2half_rn(v); }
// value not representable in storage type S (non-finite, or beyond the fp16 range)
template <typename S>
__device__ __forceinline__ bool unstorable(typename Acc<S>::T v) {
    if constexpr (sizeof(S) == 2 && !std::is_same_v<S, bf16>) return !(fabsf(v) <= 65504.f);
    else return !isfinite(v);
}
// 2^e as the compute type (GEMM output scaling of the fp16 mode; 1 elsewhere)
template <typename R>
__device__ __forceinline__ R pow2(int e) {
    return static_cast<R>(exp2f(static_cast<float>(e)));
}

// tf32 mode: a value stored for a tcgen05 consumer is rounded to the nearest
// tf32 (ties away), because kind::tf32 MMAs truncate their fp32 operands to
// tf32 - rounded once on store, the operand reaches the MMA exactly instead of
// chopped (chopping biases every product toward zero; the bias compounds along
// the contraction tree).
__device__ __forceinline__ float tf32_rn(float x) {
    uint32_t u;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(x));
    return __uint_as_float(u);
}
template <typename R>
__device__ __forceinline__ R tf32_if(R x, int32_t on) {
    if constexpr (std::is_same_v<R, float>) return on ? tf32_rn(x) : x;
    else return x;
}

// ---- leaf projection (reference project_leaf, contraction_engine.cpp:27-52,
// batched over all leaves of one level and all of their variants).
struct LeafJob {
    int64_t out_off;      // element offset of the output re-plane
    int64_t out_plane;    // elements per plane of the output buffer
    int64_t data_off;     // complex offset into the packed leaf data (double, interleaved)
    int32_t rank;         // original rank
    int32_t out_rank;     // free labels kept
    int32_t n_var;        // number of variants (>= 1)
    int32_t codes_off;    // offset into the variant code table (-1: single variant)
    // per original position p (MSB first): kind 0 free (kept), 1 pass label, 2 variant label
    int8_t kind[kMaxLeafRank];
    int16_t arg[kMaxLeafRank];  // pass: label id; variant: bit position in the group code
    int8_t obit[kMaxLeafRank];  // free: output index bit the position lands on (planned layout)
};

struct PassState {
    uint64_t slice;        // current slice index (bit b <-> sliced[b])
    uint64_t config;       // current broken-edge configuration bits
    uint32_t lo_begin, lo_end;  // finalize counts root entries with lo in [lo_begin, lo_end) (one slice: 0, 1)
};

// Pass-label source table: for a pass label, where its value comes from.
struct PassSrc {
    int8_t kind;   // 0 const, 1 slice bit, 2 config bit
    int8_t value;  // const value
    int16_t bit;
};

template <typename R>
void launch_leaf_project(const LeafJob* d_jobs, int n_jobs, const double* d_leaf_data,
                         const uint64_t* d_codes, const PassSrc* d_pass_src,
                         const PassState* d_state, R* arena, cudaStream_t st, int round_tf32 = 0);

// ---- bit-permutation transpose of a [V][2^rank] planar tensor (permute.cu).
// Output bit q (LSB=0) takes input bit src_bit[q].  Built on the host by
// make_permute(); each CTA moves tiles of up to 2^11 elements through shared
// memory so reads follow the input's contiguous runs and writes the output's,
// both as 16-byte vectors.
constexpr int kPermTileBits = 11;
struct PermuteDesc {
    int32_t rank;
    int32_t tile_bits;             // |U|: bits enumerated inside a tile
    int32_t n_outer;               // rank - tile_bits: bits enumerated across tiles
    int32_t vec;                   // 1: input bits 0,1 and output bits 0,1 are inside the tile runs
    int64_t outer_in[kMaxRank];    // input stride of outer bit j
    int64_t outer_out[kMaxRank];   // output stride of outer bit j
    int32_t in_lo[32], in_hi[64];  // input offset of tile index e (low 5 / high 6 bits)
    int32_t out_lo[32], out_hi[64];  // output offset of tile index f
    int32_t e_lo[32], e_hi[64];      // tile index e holding output element f
};
PermuteDesc make_permute(int rank, const int* src_bit);
template <typename R>
void launch_permute(const R* in, int64_t in_plane, R* out, int64_t out_plane, int64_t n_var,
                    const PermuteDesc& d, cudaStream_t st);

// ---- programmatic dependent launch (PDL).  Every kernel of a pass is launched
// with programmatic stream serialization; it waits (griddepcontrol.wait) for
// its predecessor's grid to complete -- and its memory to be visible -- before
// touching global memory, and triggers its own dependents at entry, so the
// next kernel's launch and prologue overlap this one's tail.  (The dependent
// launches only once every CTA of this grid has started.)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_enter() {
    pdl_wait();
    pdl_trigger();
}
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ---- GEMM output scatter map.  scatter == 0: row-major C.  Otherwise element
// (row m, column n) lands at
//   (m >> m_bits) * m_vstride + (n >> n_bits) * n_vstride
//     + sum_j bit_j(m) << m_pos[j] + sum_j bit_j(n) << n_pos[j]
// i.e. directly in the layout the consumer step reads (no separate permute);
// the high row / column index parts are variants folded into M / N
// (m_vstride = 0 means the dense block stride 2^(m_bits+n_bits)).
struct OutMap {
    int32_t scatter;
    int32_t m_bits, n_bits;
    int8_t m_pos[kMaxRank];
    int8_t n_pos[kMaxRank];
    int64_t m_vstride, n_vstride;
};
__host__ __device__ __forceinline__ int64_t scatter_bits(const int8_t* pos, int bits, int64_t x) {
    int64_t o = 0;
    for (int j = 0; j < bits; ++j) o |= ((x >> j) & int64_t{1}) << pos[j];
    return o;
}
// row part / column part of the output offset (additive: offset = row_off + col_off)
__host__ __device__ __forceinline__ int64_t out_row_vstride(const OutMap& om) {
    return om.m_vstride ? om.m_vstride : (int64_t{1} << (om.m_bits + om.n_bits));
}
__host__ __device__ __forceinline__ int64_t out_row_off(const OutMap& om, int64_t n_cols, int64_t m) {
    if (!om.scatter) return m * n_cols;
    return (m >> om.m_bits) * out_row_vstride(om) +
           scatter_bits(om.m_pos, om.m_bits, m & ((int64_t{1} << om.m_bits) - 1));
}
__host__ __device__ __forceinline__ int64_t out_col_off(const OutMap& om, int64_t n) {
    if (!om.scatter) return n;
    return (n >> om.n_bits) * om.n_vstride + scatter_bits(om.n_pos, om.n_bits, n & ((int64_t{1} << om.n_bits) - 1));
}

// ---- complex GEMM, both operands K-contiguous ("TN"):
//   C[v][m][n] = sum_k A[ia(v)][m][k] * B[ib(v)][n][k]
// ia / ib: device index arrays or nullptr (identity for ia, 0 for ib... see GemmArgs).
struct GemmArgs {
    const void* a;
    int64_t a_plane;   // elements per plane of A's buffer
    int64_t a_batch;   // stride between A variants (elements)
    const void* b;
    int64_t b_plane;
    int64_t b_batch;
    void* c;
    int64_t c_plane;
    int64_t c_batch;
    int64_t m, n, k;
    int64_t batch;          // number of C variants
    const int32_t* ia;      // nullptr -> A variant = v * (a_batch != 0)
    const int32_t* ib;      // nullptr -> B variant = v * (b_batch != 0)
    int32_t step;           // plan step index for the non-finite flag
    int32_t* fault;         // device flag: min step index with a non-finite output
    OutMap om;              // where C elements land inside their variant block
    int32_t scale_exp;      // outputs are stored times 2^scale_exp (fp16 per-tensor scaling; 0 otherwise)
    const int32_t* vperm;   // tcgen05 raster: result variants ordered so that runs share an operand (or nullptr)
    int32_t round_tf32;     // tf32 mode: outputs rounded to tf32 on store (see tf32_rn)
    int32_t split_tf32;     // 3xtf32 mode: fp32 operands split hi + lo on the tf32 tensor cores
};
template <typename R>
void launch_gemm_simt(const GemmArgs& g, cudaStream_t st);

// Outer-product-like steps (K <= 16): register-blocked, coalesced output writes.
bool gemm_smallk_supported(const GemmArgs& g);
template <typename R>
void launch_gemm_smallk(const GemmArgs& g, cudaStream_t st);

// Batched complex GEMV for steps with <= 4 output columns (or rows) and long K.
bool gemv_supported(const GemmArgs& g);
template <typename R>
void launch_gemv(const GemmArgs& g, cudaStream_t st);

// Fixed-order split-K reduction (W planar [split][plane][batch][m][n]) writing C
// through g.om; shared by all GEMM kernels.
template <typename S>
void launch_splitk_reduce(const typename Acc<S>::T* ws, int64_t ws_split, int splits, const GemmArgs& g,
                          cudaStream_t st);

// Slice tables: job j copies node buffer <-> table slot pext(state->slice, mask)
// (both planes, `payload` elements each).  to_table: arena -> table (build),
// else table -> arena (the per-pass gather).
struct TableJob {
    int64_t node_off, node_plane, payload;
    void* table;        // [2^popcount(mask)][2][payload] elements
    uint64_t mask;      // slice bits the node depends on
};
void launch_table_io(const TableJob* jobs, int n_jobs, const PassState* state, void* arena, int elem_bytes,
                     int to_table, cudaStream_t st);

// Scratch buffer per (stream, slot), grown on demand: slot 0 split-K partials,
// slot 1 the operand sum planes of 3M tensor-core GEMMs.
void* device_workspace(size_t bytes, cudaStream_t st, int slot = 0);
// Frees the scratch buffer of a stream that is about to be destroyed.
void release_workspace(cudaStream_t st);

// True exactly once per (flag set, current device): per-device one-time setup
// such as cudaFuncSetAttribute (a process may drive several GPUs).
bool first_on_device(std::atomic<uint64_t>& done);

// tcgen05 tensor-core path: elem 0 = fp32 storage (kind::tf32), 1 = bf16 storage
// (kind::f16 with BF16 operands); fp32 accumulation in TMEM either way.
bool gemm_tc_supported(const GemmArgs& g);
void launch_gemm_tc(const GemmArgs& g, int elem, cudaStream_t st);

// ---- finalize a pass: acc[g][i] += root[vid[g]][perm(i)]   (acc: double interleaved)
// acc[fin_g[f]][i] += sum over entries e of f (ascending batched slice lo, only
// lo in the pass's [lo_begin, lo_end)) of root[ent_vid[e]][perm(i)] * scale
template <typename R>
void launch_finalize(const R* root, int64_t root_plane, double root_scale, int64_t payload, int rank,
                     const int32_t* d_src_bit_of_canon, int n_fin, const int32_t* d_fin_g, const int32_t* d_fin_off,
                     const int32_t* d_ent_vid, const int32_t* d_ent_lo, const PassState* d_state, double* acc,
                     cudaStream_t st);

// max |value| over both planes of a float buffer (atomicMax into *out; calibration)
void launch_maxabs(const float* buf, int64_t plane, int64_t count, float* out, cudaStream_t st);

// compensated accumulation in configuration order (contraction_engine.cpp:289-302)
void launch_kahan(double* res, double* comp, const double* part, int64_t n, cudaStream_t st);
void launch_fill(double* p, double v, int64_t n, cudaStream_t st);
void launch_set_pass(PassState* d_state, uint64_t slice, uint64_t config, uint32_t lo_begin, uint32_t lo_end,
                     cudaStream_t st);

}  // namespace rcsg
