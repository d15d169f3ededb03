// Device step-program executor (host side of the contraction path).
//
// compile(): turns (network, plan, label roles) into a static program:
//   - every tree node gets a LEVEL: 0 = depends on nothing that changes, 1 =
//     depends on per-pass labels (slice / broken-edge / pinned bits), 2 =
//     depends on the candidate group (the non-open output legs); level-2 nodes
//     without pass labels form PHASE 3 (group-only), so the execution phases are
//     0 constant, 3 group-only (both cached per binding), 1 per pass, 2 per pass
//     and group;
//   - level-2 nodes are stored as [variants][payload]: one variant per DISTINCT
//     projection of the chunk's group prefixes onto the output legs inside the
//     node's subtree, so work shared by groups is done once (sparse-state
//     group batching); a step with one varying operand folds its variants into
//     M, two varying operands give a gathered batch or, for a full product with
//     separable code bits, one GEMM with the variants in M and N;
//   - each plan step is one complex GEMM whose operands are consumed K-major as
//     [kept | contracted]; layouts are planned from the root backwards and
//     every producer writes its consumer's layout through a bit-scatter map
//     (no transposes; contract_pair, contraction_engine.cpp:87-128).
// first run (group codes known): reassociate the tree for the batch (local
// rotations under a time model), rebuild, calibrate fp16 scales, bind: chunk
// capacity, first-fit arena plan over the phased schedule, slice tables for
// small per-pass subtrees, and the per-pass task DAG (lane streams, captured
// as a CUDA graph).
// run(): loops configs x slices x group chunks, accumulating canonical-order
// amplitudes per group (slices ascending, then compensated sum over configs,
// contraction_engine.cpp:241-302).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "rcsg.h"

namespace rcsg {

struct Status {
    int code = RCSG_OK;
    std::string msg;
    int step = -1;
};

// Thrown inside the library, converted to status codes at the C ABI.
struct Failure {
    int code;
    std::string msg;
    int step = -1;
};

// Sets this thread's rcsg_last_error() message and step; returns `code`
// (the C-ABI entry points of every translation unit report through it).
int record_error(int code, const std::string& msg, int step);

enum Role : int8_t { kFree = 0, kPass = 1, kVar = 2 };

struct LabelRole {
    int8_t role = kFree;
    int16_t var_bit = -1;  // kVar: bit position in the group code
    PassSrc src{};         // kPass: where the value comes from
};

struct NodeInfo {
    std::vector<int> labels;  // device layout, most significant first
    uint64_t var_mask = 0;    // group-code bits of the output legs in the subtree
    int level = 0;
    bool pass_dep = false;    // depends on slice / configuration bits
    uint64_t slice_mask = 0;  // sliced-label bits in the subtree
    bool cfg_dep = false;     // depends on broken-edge configuration bits
    bool tab = false;         // computed into slice tables once per binding (see plan_tables)
    int consumer = -1;        // program step consuming this node (-1: root)
    int64_t payload = 1;
    int64_t max_var = 1;
    int64_t off = -1;         // arena element offset of the real plane
    int64_t plane = 0;        // elements per plane (capacity)
    bool is_leaf = false;
    int64_t data_off = 0;     // leaves: complex offset into the packed leaf data
    int rank0 = 0;            // leaves: original rank
    std::vector<int> labels0; // leaves: original labels (MSB first)
};

struct StepInfo {
    int plan_index = 0;
    int a = -1, b = -1, r = -1;  // A-role operand, B-role operand, result (node ids)
    int level = 0;
    int phase = 0;  // 0 constant, 1 per pass, 2 per pass and group, 3 per group only (cached)
    bool tab = false;  // phase-1 step evaluated only while building the slice tables
    int mode = 0;  // 0 plain, 1 A-variant folded into M, 2 gathered batch
    bool perm_a = false, perm_b = false;
    PermuteDesc pa{}, pb{};
    int64_t sa_off = -1, sa_plane = 0, sb_off = -1, sb_plane = 0;  // permute scratch
    int64_t m = 1, n = 1, k = 1;
    uint64_t flops_per_variant = 0;  // 8*m*n*k
    OutMap om{};                     // epilogue scatter into the consumer's layout
};

struct ChunkData {
    std::vector<uint64_t> codes;      // per node: variant codes (concatenated)
    std::vector<int64_t> codes_off;   // per node offset into codes (-1 if level < 2)
    std::vector<int64_t> nvar;        // per node variant count
    std::vector<int32_t> idx;         // ia/ib arrays of gathered steps (concatenated)
    std::vector<int64_t> ia_off, ib_off;  // per step
    // per step: offset into idx of the result-variant order that groups the
    // variants sharing the larger operand (tcgen05 raster), -1 if none
    std::vector<int64_t> perm_off;
    // finalisation: per output group f of this chunk, its entries (root variant,
    // batched slice lo) in ascending lo
    std::vector<int32_t> fin_g, fin_off, ent_vid, ent_lo;
    // device copies
    uint64_t* d_codes = nullptr;
    int32_t* d_idx = nullptr;
    int32_t* d_fin = nullptr;  // fin_g | fin_off | ent_vid | ent_lo
    LeafJob* d_leaf_jobs = nullptr;  // phase-3 leaves first, then phase-2 leaves
    int n_leaf_jobs = 0;
    int n_leaf_jobs3 = 0;
};

class Program {
  public:
    // tf32 mode: leaves are stored rounded to tf32 like every GEMM output (tf32_rn)
    int round_leaves() const { return precision_ == RCSG_PREC_TF32 && !getenv("RCSG_TF32_CHOP") ? 1 : 0; }
    Program(const rcsg_network_desc& net, const rcsg_plan_desc& plan, const std::vector<LabelRole>& roles,
            int precision, uint64_t mem_budget);
    ~Program();
    Program(const Program&) = delete;
    Program& operator=(const Program&) = delete;

    // groups: code per group (bits at var_bit positions).  configs empty ->
    // one pass per slice with config bits 0.  d_acc: device double
    // [n_groups][2^out_rank] interleaved; accumulates (+=) the result.
    // sync == false: return once the work is enqueued on stream(); a
    // non-finite intermediate is then reported by the next synchronous call
    // or by sync().
    void run(const std::vector<uint64_t>& groups, const std::vector<uint64_t>& configs,
             uint64_t slice_begin, uint64_t slice_end, double* d_acc, rcsg_stats* stats, bool sync = true);
    void sync();

    int out_rank() const { return out_rank_; }
    void set_profile(bool on) { profile_ = on; }
    cudaStream_t stream() const { return stream_; }
    int precision() const { return precision_; }
    uint64_t plan_flops_per_pass() const { return plan_flops_; }

  private:
    void build_nodes(const rcsg_network_desc& net, const rcsg_plan_desc& plan);
    void retree(const std::vector<uint64_t>& groups);
    rcsg_network_desc stored_net();
    rcsg_plan_desc stored_plan();
    void build_steps();
    int64_t plan_arena(int64_t chunk_cap, bool assign);
    void prepare_chunks(const std::vector<uint64_t>& groups, int64_t chunk_cap);
    void bind_groups(const std::vector<uint64_t>& groups);
    void calibrate(const std::vector<uint64_t>& groups, uint64_t config, uint64_t slice);
    void exec_pass_body(int64_t P);
    // per-pass task DAG: tasks run on lane streams ordered by arena hazards,
    // so independent steps overlap (and the captured graph keeps the DAG)
    struct Task {
        int kind;  // 0 level-1 leaf projection, 1 step, 2 / 4 chunk leaf projection (phase 2 / 3),
                   // 3 chunk finalize, 6 slice-table gather
        const StepInfo* st;
        const ChunkData* ch;
    };
    void build_tasks();
    void mark_tables();
    void plan_tables();
    void build_tables();
    void free_tasks();
    void exec_pass_dag(int64_t P);
    void run_task(const Task& t, int64_t P);
    void run_pass_body(int64_t P);
    void reset_graph();
    void run_bound(size_t n_groups, const std::vector<uint64_t>& configs, uint64_t slice_begin,
                   uint64_t slice_end, double* d_acc, rcsg_stats* stats, int64_t P, int64_t acc_n, bool sync);
    void free_chunks();
    void exec_phase(int phase, const ChunkData* ch);
    void exec_step(const StepInfo& s, const ChunkData* ch);
    void* buf(int64_t off) const;
    GemmArgs step_args(const StepInfo& st, const ChunkData* ch) const;
    static int product_order(uint64_t ma, uint64_t mb, int64_t va, int64_t vb, int64_t vr);
    template <typename R>
    void exec_step_t(const StepInfo& s, const ChunkData* ch);

    int precision_;
    int elem_bytes_;
    uint64_t mem_budget_;
    std::vector<LabelRole> roles_;
    std::vector<NodeInfo> nodes_;
    std::vector<StepInfo> steps_;
    std::vector<int> root_canon_src_;  // payload bit of canonical output bit j
    std::vector<int> canon_qubit_;     // label -> open qubit (-1 if not open)
    int root_ = 0;
    int n_leaves_ = 0;
    int out_rank_ = 0;
    uint64_t plan_flops_ = 0;
    std::vector<double> leaf_data_;
    std::vector<LeafJob> static_jobs_[2];  // level 0 and level 1 leaf jobs

    // device state
    cudaStream_t stream_ = nullptr;
    cudaStream_t ls_ = nullptr;  // stream the exec_* launches go to (stream_ or a lane)
    std::vector<Task> tasks_;
    std::vector<std::vector<int>> task_wait_;  // per task: tasks on other lanes to wait for
    std::vector<int> task_lane_;
    std::vector<cudaEvent_t> task_ev_;
    std::vector<cudaStream_t> lanes_;
    std::vector<cudaEvent_t> lane_ev_;  // fork (index 0) and per-lane join events
    int n_lanes_used_ = 0;
    void* arena_ = nullptr;
    int64_t arena_elems_ = 0;
    int64_t chunk_cap_ = 0;
    double* d_leaf_data_ = nullptr;
    PassSrc* d_pass_src_ = nullptr;
    PassState* d_state_ = nullptr;
    LeafJob* d_static_jobs_[2] = {nullptr, nullptr};
    int32_t* d_canon_ = nullptr;
    int32_t* d_fault_ = nullptr;
    double* d_part_ = nullptr;   // per-config accumulator
    double* d_res_ = nullptr;
    double* d_comp_ = nullptr;
    int64_t acc_cap_ = 0;
    std::vector<ChunkData> chunks_;
    std::vector<uint64_t> bound_groups_;  // group list the chunks/arena are bound to
    // batch-aware reassociation: done once, at the first run (group codes known)
    bool tree_fixed_ = false;
    size_t n_ext_groups_ = 0;  // caller's group count of the current binding
    int64_t plan_codes_ = 0;   // distinct codes of the binding being planned (chunking test in plan_arena)
    bool level0_valid_ = false;  // level-0 (constant) results live in the arena
    bool phase3_valid_ = false;  // single chunk: its group-only (phase-3) results live in the arena
    // slice tables: small group-independent subtrees that depend on few sliced
    // labels are evaluated for every value of those labels once per binding;
    // each pass gathers the current slice's entries (one launch)
    std::vector<TableJob> tab_jobs_;
    TableJob* d_tab_jobs_ = nullptr;
    std::vector<void*> tab_mem_;
    uint64_t tab_region_mask_ = 0;
    std::vector<int> tab_boundary_;
    bool tables_valid_ = false;
    bool fault_pending_ = false; // async runs whose fault flag is not checked yet
    std::vector<int32_t> step_origin_;  // program step -> index of the plan step it came from
    // fp16 mode: per-node storage exponents (value stored times 2^-e)
    std::vector<int> node_exp_;
    bool calibrated_ = false;
    int f16_widened_ = 0;  // fp16 headroom widenings after overflow (at most 3 x 2^8)
    bool record_max_ = false;
    float* d_max_ = nullptr;
    // copies of the compile inputs (re-tree and the fp16 calibration program);
    // c_steps_ holds the steps actually executed (after reassociation)
    rcsg_network_desc calib_net_{};
    rcsg_plan_desc calib_plan_{};
    std::vector<int32_t> c_rank_, c_labels_, c_out_, c_openl_, c_openq_, c_steps_, c_sliced_, c_broken_, c_fixed_;
    cudaGraphExec_t graph_exec_ = nullptr;  // captured pass body (level 1 + chunks)
    bool graph_warm_ = false;
    uint64_t graph_launches_ = 0;
    uint64_t graph_flops_ = 0;
    uint64_t launches_ = 0;
    uint64_t exec_flops_ = 0;

    // profiling: event pairs around launches, by kernel class
    enum Cat { kCatGemmSimt = 0, kCatGemmTc = 1, kCatPermute = 2, kCatGemv = 3 };
    struct Mark {
        int cat;
        uint64_t work;
        int step;  // program step index
        int64_t m, n, k, batch;
        uint64_t bytes = 0;  // algorithmic bytes (operands + result)
    };
    bool profile_ = false;
    std::vector<cudaEvent_t> ev_pool_;
    std::vector<Mark> marks_;
    int mark_begin();
    void mark_end(int idx, int cat, uint64_t work, int step = -1, int64_t m = 0, int64_t n = 0,
                  int64_t k = 0, int64_t batch = 0);
    void collect_marks(rcsg_stats* stats);
};

}  // namespace rcsg
