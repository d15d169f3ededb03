// C ABI (include/rcsg.h) over the device executor and post-processing.
#include <climits>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "executor.hpp"
#include "postproc.hpp"
#include "rcsg.h"

using namespace rcsg;

namespace {

thread_local std::string g_msg;
thread_local int32_t g_step = -1;

template <class F>
int guard(F&& f) {
    try {
        f();
        return record_error(RCSG_OK, "", -1);
    } catch (const Failure& e) {
        return record_error(e.code, e.msg, e.step);
    } catch (const std::bad_alloc&) {
        return record_error(RCSG_ERR_CAPACITY, "host allocation failed", -1);
    } catch (const std::exception& e) {
        return record_error(RCSG_ERR_DEVICE, e.what(), -1);
    }
}

void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Failure{RCSG_ERR_DEVICE, std::string(what) + ": " + cudaGetErrorString(e)};
}

// Roles for the per-group path: every non-open qubit's output leg is a
// group-variant label with bit b = its rank among non-open qubits
// (contraction_engine.cpp:310-318); sliced / broken labels take their value
// from the pass (slice bit b <-> sliced[b], config bit b <-> broken[b],
// contraction_engine.cpp:242-248).
std::vector<LabelRole> group_roles(const rcsg_network_desc& net, const rcsg_plan_desc& plan) {
    std::vector<LabelRole> roles(net.n_labels);
    auto in_range = [&](int l) {
        if (l < 0 || l >= net.n_labels) throw Failure{RCSG_ERR_CONFIG, "plan label not in network"};
    };
    std::vector<char> open(net.n_qubits, 0);
    for (int j = 0; j < net.n_open; ++j) {
        if (net.open_qubits[j] < 0 || net.open_qubits[j] >= net.n_qubits)
            throw Failure{RCSG_ERR_CONFIG, "open qubit out of range"};
        open[net.open_qubits[j]] = 1;
    }
    int bit = 0;
    for (int q = 0; q < net.n_qubits; ++q) {
        if (open[q]) continue;
        const int l = net.output_labels[q];
        in_range(l);
        if (bit >= 64) throw Failure{RCSG_ERR_CONFIG, "more than 64 fixed qubits"};
        roles[l].role = kVar;
        roles[l].var_bit = static_cast<int16_t>(bit++);
    }
    for (int b = 0; b < plan.n_sliced; ++b) {
        in_range(plan.sliced[b]);
        LabelRole& r = roles[plan.sliced[b]];
        if (r.role != kFree) throw Failure{RCSG_ERR_CONFIG, "sliced label is also pinned otherwise"};
        r.role = kPass;
        r.src = PassSrc{1, 0, static_cast<int16_t>(b)};
    }
    for (int b = 0; b < plan.n_broken; ++b) {
        in_range(plan.broken[b]);
        LabelRole& r = roles[plan.broken[b]];
        if (r.role != kFree) throw Failure{RCSG_ERR_CONFIG, "broken label is also pinned otherwise"};
        r.role = kPass;
        r.src = PassSrc{2, 0, static_cast<int16_t>(b)};
    }
    return roles;
}

}  // namespace

int rcsg::record_error(int code, const std::string& msg, int step) {
    g_msg = msg;
    g_step = code == RCSG_OK ? -1 : step;
    return code;
}

struct rcsg_program {
    std::unique_ptr<Program> prog;
    int n_broken = 0;
    int n_sliced = 0;
    double* d_out = nullptr;  // device accumulator of rcsg_contract_groups, reused across calls
    size_t out_cap = 0;
    ~rcsg_program() {
        if (d_out) cudaFree(d_out);
    }
};

extern "C" {

const char* rcsg_last_error(int32_t* step) {
    if (step) *step = g_step;
    return g_msg.c_str();
}

int rcsg_set_device(int32_t device) {
    return guard([&] { check_cuda(cudaSetDevice(device), "cudaSetDevice"); });
}

int rcsg_compile(const rcsg_network_desc* net, const rcsg_plan_desc* plan, int32_t precision,
                 uint64_t mem_budget_bytes, rcsg_program** out) {
    return guard([&] {
        if (!net || !plan || !out) throw Failure{RCSG_ERR_CONFIG, "null argument"};
        auto p = std::make_unique<rcsg_program>();
        p->prog = std::make_unique<Program>(*net, *plan, group_roles(*net, *plan), precision, mem_budget_bytes);
        p->n_broken = plan->n_broken;
        p->n_sliced = plan->n_sliced;
        *out = p.release();
    });
}

int rcsg_compile_pinned(const rcsg_network_desc* net, const rcsg_plan_desc* plan, int32_t precision,
                        uint64_t mem_budget_bytes, const int8_t* pinned, rcsg_program** out) {
    return guard([&] {
        if (!net || !plan || !out || !pinned) throw Failure{RCSG_ERR_CONFIG, "null argument"};
        std::vector<LabelRole> roles(net->n_labels);
        for (int l = 0; l < net->n_labels; ++l) {
            if (pinned[l] < -1 || pinned[l] > 1) throw Failure{RCSG_ERR_CONFIG, "assignment values must be 0/1"};
            if (pinned[l] >= 0) {
                roles[l].role = kPass;
                roles[l].src = PassSrc{0, pinned[l], 0};
            }
        }
        for (int b = 0; b < plan->n_sliced; ++b) {
            if (plan->sliced[b] < 0 || plan->sliced[b] >= net->n_labels) throw Failure{RCSG_ERR_CONFIG, "plan label not in network"};
            roles[plan->sliced[b]].role = kPass;
            roles[plan->sliced[b]].src = PassSrc{1, 0, static_cast<int16_t>(b)};
        }
        for (int b = 0; b < plan->n_broken; ++b) {
            if (plan->broken[b] < 0 || plan->broken[b] >= net->n_labels) throw Failure{RCSG_ERR_CONFIG, "plan label not in network"};
            roles[plan->broken[b]].role = kPass;
            roles[plan->broken[b]].src = PassSrc{2, 0, static_cast<int16_t>(b)};
        }
        auto p = std::make_unique<rcsg_program>();
        p->prog = std::make_unique<Program>(*net, *plan, roles, precision, mem_budget_bytes);
        p->n_broken = plan->n_broken;
        p->n_sliced = plan->n_sliced;
        *out = p.release();
    });
}

int rcsg_program_free(rcsg_program* prog) {
    return guard([&] { delete prog; });
}

int rcsg_program_stream(rcsg_program* prog, void** out) {
    return guard([&] {
        if (!prog || !out) throw Failure{RCSG_ERR_CONFIG, "null argument"};
        *out = static_cast<void*>(prog->prog->stream());
    });
}

int rcsg_program_set_profile(rcsg_program* prog, int32_t on) {
    return guard([&] {
        if (!prog) throw Failure{RCSG_ERR_CONFIG, "null program"};
        prog->prog->set_profile(on != 0);
    });
}

int rcsg_contract_groups_device(rcsg_program* prog, uint64_t n_groups, const uint64_t* group_fixed,
                                uint64_t n_configs, const uint64_t* configs, uint64_t slice_begin,
                                uint64_t slice_end, double* d_acc, int32_t sync, rcsg_stats* stats) {
    return guard([&] {
        if (!prog) throw Failure{RCSG_ERR_CONFIG, "null program"};
        if (n_groups < 1) throw Failure{RCSG_ERR_CONFIG, "group count must be >= 1"};
        if (n_configs == 0 && prog->n_broken > 0)
            throw Failure{RCSG_ERR_CONFIG, "plan has broken edges; exact contraction needs a plan without them"};
        if (n_configs > 0 && prog->n_broken == 0)
            throw Failure{RCSG_ERR_CONFIG, "broken-edge labels do not match the plan"};
        if (slice_end > (uint64_t{1} << prog->n_sliced) || slice_begin >= slice_end)
            throw Failure{RCSG_ERR_CONFIG, "slice range outside [0, 2^|sliced|)"};
        std::vector<uint64_t> groups(group_fixed, group_fixed + n_groups);
        std::vector<uint64_t> cfgs(configs, configs + n_configs);
        prog->prog->run(groups, cfgs, slice_begin, slice_end, d_acc, stats, sync != 0);
    });
}

int rcsg_program_sync(rcsg_program* prog) {
    return guard([&] {
        if (!prog) throw Failure{RCSG_ERR_CONFIG, "null program"};
        prog->prog->sync();
    });
}

int rcsg_contract_groups(rcsg_program* prog, uint64_t n_groups, const uint64_t* group_fixed,
                         uint64_t n_configs, const uint64_t* configs, uint64_t slice_begin,
                         uint64_t slice_end, double* out_amps, rcsg_stats* stats) {
    return guard([&] {
        if (!prog) throw Failure{RCSG_ERR_CONFIG, "null program"};
        const size_t n = static_cast<size_t>(n_groups) << prog->prog->out_rank();
        if (prog->out_cap < std::max<size_t>(n, 1)) {  // grow-only; the program's stream orders its reuse
            if (prog->d_out) {
                check_cuda(cudaStreamSynchronize(prog->prog->stream()), "cudaStreamSynchronize");
                cudaFree(prog->d_out);
                prog->d_out = nullptr;
                prog->out_cap = 0;
            }
            check_cuda(cudaMalloc(&prog->d_out, std::max<size_t>(n, 1) * 2 * sizeof(double)), "cudaMalloc");
            prog->out_cap = std::max<size_t>(n, 1);
        }
        double* d = prog->d_out;
        // zero on the program's (non-blocking) stream: the accumulation below is
        // ordered after it without a device-wide synchronisation
        check_cuda(cudaMemsetAsync(d, 0, n * 2 * sizeof(double), prog->prog->stream()), "cudaMemsetAsync");
        const int rc = rcsg_contract_groups_device(prog, n_groups, group_fixed, n_configs, configs,
                                                   slice_begin, slice_end, d, 1, stats);
        if (rc) throw Failure{rc, g_msg, g_step};
        check_cuda(cudaMemcpy(out_amps, d, n * 2 * sizeof(double), cudaMemcpyDeviceToHost), "cudaMemcpy");
    });
}

int rcsg_execute_assignment(const rcsg_network_desc* net, const rcsg_plan_desc* plan, int32_t precision,
                            const int8_t* assign, double* out, uint64_t* n_out) {
    return guard([&] {
        if (!net || !plan || !assign) throw Failure{RCSG_ERR_CONFIG, "null argument"};
        std::vector<LabelRole> roles(net->n_labels);
        for (int l = 0; l < net->n_labels; ++l) {
            if (assign[l] < -1 || assign[l] > 1) throw Failure{RCSG_ERR_CONFIG, "assignment values must be 0/1"};
            if (assign[l] >= 0) {
                roles[l].role = kPass;
                roles[l].src = PassSrc{0, assign[l], 0};
            }
        }
        Program prog(*net, *plan, roles, precision, 0);
        const size_t n = size_t{1} << prog.out_rank();
        double* d = nullptr;
        check_cuda(cudaMalloc(&d, n * 2 * sizeof(double)), "cudaMalloc");
        std::unique_ptr<double, decltype(&cudaFree)> hold(d, &cudaFree);
        check_cuda(cudaMemsetAsync(d, 0, n * 2 * sizeof(double), prog.stream()), "cudaMemsetAsync");
        prog.run({0}, {}, 0, 1, d, nullptr);
        if (out) check_cuda(cudaMemcpy(out, d, n * 2 * sizeof(double), cudaMemcpyDeviceToHost), "cudaMemcpy");
        if (n_out) *n_out = n;
    });
}

int rcsg_topk(const rcsg_candidates* cs, const double* d_amps, uint64_t k, uint64_t* out) {
    return guard([&] { topk_select(*cs, d_amps, true, k, out, 0); });
}

int rcsg_topk_probs(const rcsg_candidates* cs, const double* d_probs, uint64_t k, uint64_t* out) {
    return guard([&] { topk_select(*cs, d_probs, false, k, out, 0); });
}

int rcsg_direct_sample(const rcsg_candidates* cs, const double* d_amps, uint64_t rng_seed, uint64_t* out) {
    return guard([&] { direct_sample(*cs, d_amps, true, rng_seed, out, 0); });
}

int rcsg_direct_sample_probs(const rcsg_candidates* cs, const double* d_probs, uint64_t rng_seed,
                             uint64_t* out) {
    return guard([&] { direct_sample(*cs, d_probs, false, rng_seed, out, 0); });
}

int rcsg_xeb(int32_t n_qubits, uint64_t count, const double* q, double* out) {
    return guard([&] {
        if (count == 0) throw Failure{RCSG_ERR_CONFIG, "XEB needs at least one sample"};
        if (!q || !out) throw Failure{RCSG_ERR_CONFIG, "null argument"};
        // host q (the reference's ProbFn values): staged to the device and reduced there
        double* d = nullptr;
        check_cuda(cudaMalloc(&d, count * sizeof(double)), "cudaMalloc");
        std::unique_ptr<double, decltype(&cudaFree)> hold(d, &cudaFree);
        check_cuda(cudaMemcpy(d, q, count * sizeof(double), cudaMemcpyHostToDevice), "cudaMemcpy");
        *out = xeb_device(n_qubits, count, nullptr, nullptr, d);
    });
}

int rcsg_xeb_state(int32_t n_qubits, uint64_t count, const uint64_t* indices, const double* d_state, double* out) {
    return guard([&] {
        if (!indices || !d_state || !out) throw Failure{RCSG_ERR_CONFIG, "null argument"};
        for (uint64_t i = 0; i < count; ++i)
            if (n_qubits < 64 && (indices[i] >> n_qubits) != 0)
                throw Failure{RCSG_ERR_CONFIG, "sample index outside the statevector"};
        *out = xeb_device(n_qubits, count, d_state, indices, nullptr);
    });
}

int rcsg_postprocess(const rcsg_candidates* cs, const double* d_amps, uint64_t k, uint64_t* out_topk,
                     int32_t direct, uint64_t rng_seed, uint64_t* out_direct, const double* d_state,
                     rcsg_post_stats* stats) {
    return guard([&] {
        if (!cs || !d_amps) throw Failure{RCSG_ERR_CONFIG, "null argument"};
        if (direct && !out_direct) throw Failure{RCSG_ERR_CONFIG, "direct sampling needs an output buffer"};
        const char* e = getenv("RCSG_TOPK_PATH");
        const PostResult r = postprocess(*cs, d_amps, true, k, out_topk, direct != 0, rng_seed, out_direct, d_state,
                                         false, e ? atoi(e) : 0);
        if (stats) {
            stats->device_ms = r.device_ms;
            stats->bytes = r.bytes;
            stats->candidates_kept = r.candidates_kept;
            stats->fast_path = r.fast_path ? 1 : 0;
            stats->fallback = r.fallback ? 1 : 0;
            stats->xeb_topk = r.xeb_top;
            stats->xeb_direct = r.xeb_direct;
        }
    });
}

int rcsg_device_alloc(uint64_t bytes, void** out) {
    return guard([&] { check_cuda(cudaMalloc(out, std::max<uint64_t>(bytes, 1)), "cudaMalloc"); });
}

int rcsg_device_free(void* p) {
    return guard([&] { check_cuda(cudaFree(p), "cudaFree"); });
}

int rcsg_memcpy(void* dst, const void* src, uint64_t bytes, int32_t kind) {
    return guard([&] {
        const cudaMemcpyKind k = kind == 1 ? cudaMemcpyHostToDevice
                                 : kind == 2 ? cudaMemcpyDeviceToHost
                                             : cudaMemcpyDeviceToDevice;
        check_cuda(cudaMemcpy(dst, src, bytes, k), "cudaMemcpy");
    });
}

}  // extern "C"
