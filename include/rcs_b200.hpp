// rcs_b200.hpp — C++ host API of the B200-native sampler (namespace rcs).
//
// Drop-in surface for the reference's hot path (/root/reference/proj/include/rcs):
// same type names, field meanings, function signatures, result semantics and
// exception types, so a caller of the reference's
//   contract / contract_group / execute_assignment   (contraction_engine.hpp:54-76)
//   top_k_select / direct_sample / xeb               (sampling.hpp:42-51)
// switches by including this header and linking libpaper_2406_18889_b200.so.
// The inputs to that path (circuit, network, plan, candidate set) are
// re-implemented host-side with identical semantics so plans and candidate sets
// are bit-identical to the reference's.  Contraction and post-processing run on
// the GPU through the C ABI in rcsg.h; there is no CPU execution path.
#pragma once

#include <complex>
#include <cstdint>
#include <functional>
#include <map>
#include <span>
#include <stdexcept>
#include <iosfwd>
#include <string>
#include <utility>
#include <vector>

namespace rcs {

using cplx = std::complex<double>;
using Label = int;

// ---- errors (reference errors.hpp:9-25; exit codes 2/3/4)
struct Error : std::runtime_error {
    Error(std::string msg, int code) : std::runtime_error(std::move(msg)), exit_code(code) {}
    int exit_code;
};
struct ConfigError : Error {
    explicit ConfigError(std::string msg) : Error(std::move(msg), 2) {}
};
struct NumericFault : Error {
    NumericFault(std::string msg, int step) : Error(std::move(msg), 3), step_index(step) {}
    int step_index;
};
struct CapacityError : Error {
    explicit CapacityError(std::string msg) : Error(std::move(msg), 4) {}
};
// CUDA / NCCL runtime failure (C-ABI status 5; CLI exit 1).
struct DeviceError : Error {
    explicit DeviceError(std::string msg) : Error(std::move(msg), 1) {}
};

// ---- SplitMix64 stream (reference rng.hpp:10-45); counter-based form in rcs_rng.h
class Rng {
  public:
    explicit Rng(std::uint64_t seed) : s_(seed) {}
    std::uint64_t next_u64();
    double next_double();
    std::uint64_t next_below(std::uint64_t bound);
    bool next_bool() { return (next_u64() >> 63) != 0; }
    Rng split(std::uint64_t tag) const;
    std::uint64_t state() const { return s_; }

  private:
    std::uint64_t s_;
};

// ---- circuit (reference circuit.hpp:13-63)
enum class GateKind { SqrtX, SqrtY, SqrtW, TwoQubit };
const char* gate_kind_name(GateKind kind);
GateKind gate_kind_from_name(const std::string& name);
std::vector<cplx> gate_unitary(GateKind kind);

struct Gate {
    GateKind kind;
    std::vector<int> targets;
    std::vector<cplx> unitary;
    int matrix_dim() const { return targets.size() == 1 ? 2 : 4; }
};
struct Layer {
    std::vector<Gate> gates;
};
struct Circuit {
    int n_qubits = 0;
    std::uint64_t seed = 0;
    std::string topology;
    std::vector<Layer> layers;
    bool exceeds_exact_cap = false;
    int n_cycles() const { return static_cast<int>(layers.size()) / 2; }
};
struct Topology {
    std::string name;
    int n_qubits = 0;
    std::vector<std::vector<std::pair<int, int>>> patterns;
    std::vector<int> sequence;
};
// "line", "ring", "grid(R,C)" as in the reference, plus (new) "sycamore53" and
// "zuchongzhi60" (diagonal lattices of 9 x 6 sites minus one, and 10 x 6).
Topology make_topology(const std::string& name, int n_qubits);
Circuit gen_random_circuit(int n_qubits, int n_cycles, const std::string& topology,
                           std::uint64_t seed);

// ---- tensor network (reference tensor_network.hpp:12-48)
struct Tensor {
    std::vector<Label> labels;  // labels[0] is the most significant index bit
    std::vector<cplx> data;
    int rank() const { return static_cast<int>(labels.size()); }
    std::uint64_t size() const { return data.size(); }
};
struct WireEdge {
    Label label;
    int qubit;
    int layer;
};
struct TensorNetwork {
    std::vector<Tensor> tensors;
    std::vector<std::string> label_names;
    std::vector<Label> output_labels;
    std::vector<Label> open_labels;
    std::vector<int> open_qubits;
    std::vector<WireEdge> wire_edges;
    int n_qubits = 0;
    int n_layers = 0;
    const std::string& label_name(Label l) const { return label_names[l]; }
    Label label_by_name(const std::string& name) const;
    bool is_open(Label l) const;
};
TensorNetwork circuit_to_network(const Circuit& circuit, const std::vector<int>& open_qubits);

// ---- contraction plan (reference contraction_plan.hpp:11-74)
struct PlanStep {
    int lhs = -1, rhs = -1, result = -1;
    std::vector<Label> result_labels;  // sorted ascending (not the executor layout)
    std::uint64_t summed = 0;
    std::uint64_t flops = 0;  // 8 real FLOPs per complex multiply-add
    std::uint64_t result_bytes = 0;
};
struct ContractionPlan {
    std::vector<PlanStep> steps;
    std::vector<Label> sliced;
    std::vector<Label> broken;
    std::vector<Label> fixed_outputs;
    std::uint64_t flops_per_slice = 0;
    std::uint64_t traffic_bytes_per_slice = 0;
    std::uint64_t peak_bytes = 0;
    std::uint64_t memory_budget_bytes = 0;
    std::uint64_t n_slices() const { return std::uint64_t{1} << sliced.size(); }
    std::uint64_t subtask_flops() const { return flops_per_slice * n_slices(); }
    std::uint64_t subtask_traffic_bytes() const { return traffic_bytes_per_slice * n_slices(); }
};
enum class SearchEffort { Low, Medium, High };
ContractionPlan find_contraction_path(const TensorNetwork& network,
                                      std::uint64_t memory_budget_bytes,
                                      SearchEffort effort = SearchEffort::Medium,
                                      std::uint64_t seed = 0,
                                      const std::vector<Label>& broken = {});
std::vector<Label> select_broken_edges(const TensorNetwork& network, int k_edges,
                                       std::uint64_t seed = 0);

// ---- planner at scale (new) -------------------------------
// find_contraction_path dispatches on the planner kind:
//   Reference - the reference algorithm restated bit for bit (contraction_plan.cpp:85-377);
//   Scale     - log-domain, batch-aware, randomized-greedy + subtree-reconfiguration
//               planner with stem-aware slicing (planner_scale.cpp);
//   Auto      - (default) Reference wherever it works, Scale where the reference's
//               uint64 costs overflow (rank >= 60) or its budget slicing stalls.
enum class PlannerKind { Reference, Scale, Auto };
struct ScalePlannerOptions {
    std::uint64_t n_groups = 1;  // group batch the costs model (variant counts min(M, 2^b))
    int trials = 0;              // hyper-optimisation trials (0: 256 / 1024 / 4096 by effort)
    int threads = 0;             // host threads (0: all)
    int refine = 16;             // best trees refined by subtree reconfiguration
    int phases = 1;              // 2: search again on the network with phase 1's slice set cut
};
struct ScalePlanReport {
    double log2_total_flops = 0;              // all slices, batched cost model
    double log2_flops_per_slice_batched = 0;  // slice-dependent steps, one slice
    double log2_flops_once_batched = -1;      // slice-independent steps (run once)
    double log2_max_size = 0;                 // widest tensor incl. variant bits
    double seconds = 0;
    int n_sliced = 0, trials = 0, winning_trial = -1, threads = 0, reduced_tensors = 0;
};
void set_planner(PlannerKind kind, const ScalePlannerOptions& options = {});
PlannerKind get_planner();
ContractionPlan find_contraction_path_reference(const TensorNetwork& network, std::uint64_t memory_budget_bytes,
                                                SearchEffort effort, std::uint64_t seed,
                                                const std::vector<Label>& broken);
ContractionPlan find_contraction_path_scale(const TensorNetwork& network, std::uint64_t memory_budget_bytes,
                                            SearchEffort effort, std::uint64_t seed,
                                            const std::vector<Label>& broken = {},
                                            const ScalePlannerOptions& options = {},
                                            ScalePlanReport* report = nullptr);
// True when the reference planner's greedy tree already saturates its uint64
// costs, i.e. Auto hands the network to the scale planner.
bool reference_planner_overflows(const TensorNetwork& network, const std::vector<Label>& broken = {});

// ---- executor (reference contraction_engine.hpp:13-86)
struct BrokenEdgeConfig {
    std::vector<Label> broken_labels;
    std::vector<std::uint64_t> configurations;
    int k() const { return static_cast<int>(broken_labels.size()); }
    std::uint64_t m() const { return configurations.size(); }
    double predicted_fidelity() const;
};
BrokenEdgeConfig make_broken_config(std::vector<Label> broken_labels, std::uint64_t m,
                                    std::uint64_t seed);

struct ExecutionStats {
    std::uint64_t flops = 0;       // plan-equivalent FLOPs (8 per complex MAC)
    std::uint64_t peak_bytes = 0;  // device arena bytes
};
struct SubtaskTiming {
    std::uint64_t subtask_id = 0;
    std::uint64_t config_bits = 0;
    double wall_ms = 0;
    std::uint64_t flops = 0;
};
struct AmplitudeBatch {
    std::uint64_t group_id = 0;
    int n_open = 0;
    std::uint64_t fixed_bits = 0;
    std::vector<cplx> amplitudes;
};
struct ContractResult {
    std::vector<cplx> amplitudes;
    std::vector<SubtaskTiming> timings;
    ExecutionStats stats;
};

std::vector<cplx> execute_assignment(const TensorNetwork& network, const ContractionPlan& plan,
                                     const std::map<Label, int>& assignment,
                                     ExecutionStats* stats = nullptr);
// Device context (new): one process drives these local GPUs (rcsg_init; NCCL
// over NVLink).  With a context, contract() shards the slices of a
// group-shaped pin set (every non-open output pinned, as contract_group does)
// over min(workers, devices) GPUs; the result never depends on `workers`
// (canonical slice blocks summed in block order).  Without one, `workers` is
// accepted for signature compatibility and one GPU runs.  An empty list
// releases the context.
void init_devices(const std::vector<int>& devices);
int device_count();
// Compiled device programs are cached per (network, plan, precision, pins),
// LRU over 8 entries; this frees them.
void clear_program_cache();
ContractResult contract(const TensorNetwork& network, const ContractionPlan& plan,
                        const BrokenEdgeConfig* config,
                        const std::map<Label, int>& fixed_outputs = {}, int workers = 1);
AmplitudeBatch contract_group(const TensorNetwork& network, const ContractionPlan& plan,
                              const BrokenEdgeConfig* config, std::uint64_t group_id,
                              std::uint64_t fixed_bits);
// Group-batched production path (new): amplitudes of every group, [M][2^l].
std::vector<AmplitudeBatch> contract_groups(const TensorNetwork& network,
                                            const ContractionPlan& plan,
                                            const BrokenEdgeConfig* config,
                                            const std::vector<std::uint64_t>& group_fixed);

struct FidelityResult {
    double value = 0;
    bool zero_norm_warning = false;
};
FidelityResult state_fidelity(std::span<const cplx> approx, std::span<const cplx> exact);

// ---- exact statevector (reference statevector.hpp), computed on the GPU
// (rcsg_statevector: bit-identical to the reference's complex<double> gate loop).
// Qubit q maps to bit q of the array index.
struct StateVector {
    int n_qubits = 0;
    std::vector<cplx> amps;
    double norm_sq() const;
};
constexpr int kDefaultExactCap = 24;
// Throws CapacityError above `cap` qubits (the host copy is 16 B x 2^n).
StateVector simulate_exact(const Circuit& circuit, int cap = kDefaultExactCap);
double ideal_probability(const StateVector& state, const std::string& bitstring);
std::uint64_t bitstring_to_index(const std::string& bitstring);
std::string index_to_bitstring(std::uint64_t index, int n_qubits);
// Binary amplitude dump (reference format): 16-byte header {"QSVD", version u32 = 1,
// n_qubits u32, pad u32}, then little-endian float64 (re, im) interleaved.
void dump_amplitudes(const StateVector& state, std::ostream& out);
StateVector load_amplitudes(std::istream& in);

// Precision of the device executor: "f64" (default; reference-grade), "f32",
// "tf32" (tcgen05 tensor cores), "3xtf32" (fp32-grade accuracy on the tf32 tensor
// cores: fp32 operands split into hi + lo halves, three products per real product),
// "bf16", "f16" (fp16 storage with per-tensor power-of-two scales).
void set_precision(const std::string& precision);
std::string get_precision();

// ---- sampler (reference sampling.hpp:10-85)
using ProbFn = std::function<double(std::uint64_t)>;
struct CandidateSet {
    int n_qubits = 0;
    std::vector<int> open_qubits;
    std::vector<std::uint64_t> group_fixed;
    int duplicate_groups = 0;
    int l() const { return static_cast<int>(open_qubits.size()); }
    std::uint64_t n_groups() const { return group_fixed.size(); }
    std::uint64_t size() const { return n_groups() << l(); }
    std::uint64_t member(std::uint64_t group, std::uint64_t i) const;
};
CandidateSet build_candidate_set(int n_qubits, std::vector<int> open_qubits,
                                 std::uint64_t n_groups, std::uint64_t seed);
enum class Provenance { Direct, TopK };
struct SampleSet {
    int n_qubits = 0;
    std::vector<std::uint64_t> bitstrings;
    Provenance provenance = Provenance::Direct;
    std::uint64_t k = 0;
};
double xeb(const SampleSet& samples, const ProbFn& q);
SampleSet top_k_select(const CandidateSet& candidates, const ProbFn& p, std::uint64_t k);
SampleSet direct_sample(const CandidateSet& candidates, const ProbFn& p, std::uint64_t rng_seed);
double predicted_topk_xeb(double fidelity, std::uint64_t candidate_size, std::uint64_t k);

// ---- artifact formats (reference writers, byte-compatible)
// plan.json (contraction_plan.cpp:451-491) and its import: the post-order steps
// are rebuilt from the nested "order" pairs, sliced / broken from label names.
std::string plan_to_json(const ContractionPlan& plan, const TensorNetwork& network);
ContractionPlan plan_from_json(const std::string& json, const TensorNetwork& network);
// timings.csv (contraction_engine.cpp:347-354)
std::string timings_to_csv(const std::vector<SubtaskTiming>& timings);
// samples.txt (sampling.cpp:177-210): character q = qubit q
std::string samples_to_text(const SampleSet& samples);
SampleSet samples_from_text(const std::string& text);
// metrics.json (harness.cpp:154-175, schema "rcs-metrics-v1")
struct MetricsReport {
    double xeb = 0, fidelity = 0, predicted_xeb = 0, pearson_r = 0;
    double pt_ks_statistic = 0, pt_p_value = 0, xeb_over_fidelity = 0;
};
struct MetricsInputs {
    int n_qubits = 0, n_cycles = 0;
    std::string topology;
    std::uint64_t seed = 0;
    std::size_t l = 0;
    std::uint64_t n_groups = 0;
    int broken_edges = 0;
    std::uint64_t m_configs = 1, k = 0;
    std::string sample_mode = "top_k";  // "direct" | "top_k"
};
std::string metrics_to_json(const MetricsReport& metrics, const MetricsInputs& inputs);
std::uint64_t lexicographic_key(std::uint64_t index, int n_qubits);

}  // namespace rcs
