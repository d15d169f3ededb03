// Flat C entry points over the host C++ API (rcsh_*), for FFI callers that are
// not C++ (the Python package binds these and rcsg.h with ctypes).  Each one
// wraps the rcs:: call named in its comment; the hot-path calls end in the
// device C ABI (rcsg.h).
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <unordered_map>

#include "flat.hpp"
#include "rcs_b200.hpp"
#include "rcsg.h"

using namespace rcs;

namespace {

thread_local std::string g_err;
thread_local int g_step = -1;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const NumericFault& e) {
        g_err = e.what();
        g_step = e.step_index;
        return e.exit_code;
    } catch (const DeviceError& e) {
        g_err = e.what();
        return RCSG_ERR_DEVICE;
    } catch (const Error& e) {
        g_err = e.what();
        return e.exit_code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return RCSG_ERR_DEVICE;
    }
}

[[noreturn]] void raise_rcsg(int rc) {
    int32_t step = -1;
    const std::string msg = rcsg_last_error(&step);
    if (rc == RCSG_ERR_CONFIG) throw ConfigError(msg);
    if (rc == RCSG_ERR_NUMERIC) throw NumericFault(msg, step);
    if (rc == RCSG_ERR_CAPACITY) throw CapacityError(msg);
    throw DeviceError(msg);
}

struct Handle {
    Circuit circuit;
    TensorNetwork net;
    ContractionPlan plan;
    BrokenEdgeConfig config;
    bool has_config = false;
    std::unique_ptr<Flat> flat;
    std::map<std::pair<int, std::uint64_t>, rcsg_program*> programs;
    bool profile = false;
    ~Handle() {
        for (auto& [k, p] : programs) rcsg_program_free(p);
    }
    rcsg_program* program(int precision, std::uint64_t budget) {
        auto key = std::make_pair(precision, budget);
        auto it = programs.find(key);
        rcsg_program* p = nullptr;
        if (it != programs.end()) {
            p = it->second;
        } else {
            if (!flat) flat = flatten(net, plan);
            if (int rc = rcsg_compile(&flat->net, &flat->plan, precision, budget, &p)) raise_rcsg(rc);
            programs[key] = p;
        }
        rcsg_program_set_profile(p, profile ? 1 : 0);
        return p;
    }
};

SearchEffort effort_of(int e) {
    return e == 0 ? SearchEffort::Low : (e == 2 ? SearchEffort::High : SearchEffort::Medium);
}

void copy_amps(const std::vector<cplx>& v, double* out) {
    for (std::size_t i = 0; i < v.size(); ++i) {
        out[2 * i] = v[i].real();
        out[2 * i + 1] = v[i].imag();
    }
}

ProbFn prob_map(const CandidateSet& cs, const double* probs) {
    auto map = std::make_shared<std::unordered_map<std::uint64_t, double>>();
    const std::uint64_t per = std::uint64_t{1} << cs.l();
    for (std::uint64_t g = 0; g < cs.n_groups(); ++g)
        for (std::uint64_t i = 0; i < per; ++i) (*map)[cs.member(g, i)] = probs[g * per + i];
    return [map](std::uint64_t idx) {
        auto it = map->find(idx);
        return it == map->end() ? -1.0 : it->second;
    };
}

CandidateSet make_set(int n, const int* open, int l, std::uint64_t n_groups, const std::uint64_t* fixed) {
    CandidateSet cs;
    cs.n_qubits = n;
    cs.open_qubits.assign(open, open + l);
    cs.group_fixed.assign(fixed, fixed + n_groups);
    return cs;
}

}  // namespace

extern "C" {

const char* rcsh_last_error(int* step) {
    if (step) *step = g_step;
    return g_err.c_str();
}

// gen_random_circuit -> circuit_to_network(open) -> select_broken_edges ->
// find_contraction_path -> make_broken_config (the per-group pipeline).
int rcsh_build(int n, int cycles, const char* topology, std::uint64_t seed, const int* open, int n_open,
               std::uint64_t budget, int effort, int k_broken, std::uint64_t m, void** out) {
    return guarded([&] {
        auto h = std::make_unique<Handle>();
        h->circuit = gen_random_circuit(n, cycles, topology, seed);
        h->net = circuit_to_network(h->circuit, std::vector<int>(open, open + n_open));
        std::vector<Label> broken;
        if (k_broken > 0) broken = select_broken_edges(h->net, k_broken, seed);
        h->plan = find_contraction_path(h->net, budget, effort_of(effort), seed, broken);
        if (k_broken > 0) {
            h->config = make_broken_config(broken, m, seed);
            h->has_config = true;
        }
        *out = h.release();
    });
}

// Same pipeline with an explicit planner: planner 0 reference, 1 scale, 2 auto,
// 3 none (the plan is imported next with rcsh_plan_import);
// n_groups / trials / threads tune the scale planner (ScalePlannerOptions).
// report (may be null): [log2 total flops, log2 per-slice flops (batched model),
// log2 once-only flops, log2 widest tensor, seconds, n_sliced, trials,
// winning trial, threads, reduced tensors] - filled when the scale planner ran.
int rcsh_build_ex(int n, int cycles, const char* topology, std::uint64_t seed, const int* open, int n_open,
                  std::uint64_t budget, int effort, int k_broken, std::uint64_t m, int planner,
                  std::uint64_t n_groups, int trials, int threads, double* report, void** out) {
    return guarded([&] {
        auto h = std::make_unique<Handle>();
        h->circuit = gen_random_circuit(n, cycles, topology, seed);
        h->net = circuit_to_network(h->circuit, std::vector<int>(open, open + n_open));
        std::vector<Label> broken;
        if (k_broken > 0) broken = select_broken_edges(h->net, k_broken, seed);
        ScalePlannerOptions opt;
        opt.n_groups = n_groups ? n_groups : 1;
        opt.trials = trials;
        opt.threads = threads;
        ScalePlanReport rep;
        bool scale = planner == 1 || (planner == 2 && reference_planner_overflows(h->net, broken));
        if (planner == 3) {
            scale = false;  // no planning: the caller imports a plan file next (rcsh_plan_import)
        } else if (planner == 0) {
            h->plan = find_contraction_path_reference(h->net, budget, effort_of(effort), seed, broken);
        } else if (scale) {
            h->plan = find_contraction_path_scale(h->net, budget, effort_of(effort), seed, broken, opt, &rep);
        } else {
            try {
                h->plan = find_contraction_path_reference(h->net, budget, effort_of(effort), seed, broken);
            } catch (const ConfigError& e) {
                if (std::string(e.what()).rfind("cannot slice below memory budget", 0) != 0) throw;
                h->plan = find_contraction_path_scale(h->net, budget, effort_of(effort), seed, broken, opt, &rep);
                scale = true;
            }
        }
        if (report) {
            const double r[10] = {rep.log2_total_flops, rep.log2_flops_per_slice_batched, rep.log2_flops_once_batched,
                                  rep.log2_max_size, rep.seconds, static_cast<double>(rep.n_sliced),
                                  static_cast<double>(rep.trials), static_cast<double>(rep.winning_trial),
                                  static_cast<double>(rep.threads), static_cast<double>(rep.reduced_tensors)};
            for (int i = 0; i < 10; ++i) report[i] = scale ? r[i] : -1.0;
        }
        if (k_broken > 0) {
            h->config = make_broken_config(broken, m, seed);
            h->has_config = true;
        }
        *out = h.release();
    });
}

// Hand-built network (names '\n'-separated) planned with find_contraction_path.
int rcsh_build_network(int n_leaves, const int* leaf_rank, const int* leaf_labels, const double* leaf_data,
                       const char* names, int n_qubits, const int* output_labels, int n_open,
                       const int* open_labels, const int* open_qubits, std::uint64_t budget, int effort,
                       std::uint64_t seed, int n_broken, const int* broken, void** out) {
    return guarded([&] {
        auto h = std::make_unique<Handle>();
        TensorNetwork& net = h->net;
        std::string all(names);
        for (std::size_t a = 0; a < all.size();) {
            const std::size_t b = all.find('\n', a);
            net.label_names.push_back(all.substr(a, b - a));
            if (b == std::string::npos) break;
            a = b + 1;
        }
        std::size_t lo = 0, dof = 0;
        for (int t = 0; t < n_leaves; ++t) {
            Tensor tt;
            tt.labels.assign(leaf_labels + lo, leaf_labels + lo + leaf_rank[t]);
            const std::size_t sz = std::size_t{1} << leaf_rank[t];
            for (std::size_t i = 0; i < sz; ++i)
                tt.data.emplace_back(leaf_data[2 * (dof + i)], leaf_data[2 * (dof + i) + 1]);
            lo += leaf_rank[t];
            dof += sz;
            net.tensors.push_back(std::move(tt));
        }
        net.n_qubits = n_qubits;
        net.output_labels.assign(output_labels, output_labels + n_qubits);
        net.open_labels.assign(open_labels, open_labels + n_open);
        net.open_qubits.assign(open_qubits, open_qubits + n_open);
        h->plan = find_contraction_path(net, budget, effort_of(effort), seed,
                                        std::vector<Label>(broken, broken + n_broken));
        *out = h.release();
    });
}

void rcsh_free(void* h) { delete static_cast<Handle*>(h); }

void rcsh_set_profile(void* h, int on) { static_cast<Handle*>(h)->profile = on != 0; }

// Frees the handle's compiled programs (their device arenas); the next call compiles again.
void rcsh_release_programs(void* hp) {
    Handle* h = static_cast<Handle*>(hp);
    for (auto& [k, p] : h->programs) rcsg_program_free(p);
    h->programs.clear();
}

// Stream of the handle's compiled program for (precision, budget); compiles it if needed.
int rcsh_program_stream(void* hp, int precision, std::uint64_t budget, void** out) {
    return guarded([&] {
        rcsg_program* p = static_cast<Handle*>(hp)->program(precision, budget);
        if (int rc = rcsg_program_stream(p, out)) raise_rcsg(rc);
    });
}

void rcsh_net_sizes(void* hp, std::int64_t* sizes) {
    const Handle* h = static_cast<Handle*>(hp);
    std::int64_t sum_rank = 0, sum_amps = 0;
    for (const Tensor& t : h->net.tensors) {
        sum_rank += t.rank();
        sum_amps += static_cast<std::int64_t>(t.data.size());
    }
    sizes[0] = static_cast<std::int64_t>(h->net.tensors.size());
    sizes[1] = static_cast<std::int64_t>(h->net.label_names.size());
    sizes[2] = h->net.n_qubits;
    sizes[3] = static_cast<std::int64_t>(h->net.open_labels.size());
    sizes[4] = sum_rank;
    sizes[5] = sum_amps;
    sizes[6] = h->net.n_layers;
    sizes[7] = static_cast<std::int64_t>(h->net.wire_edges.size());
}

void rcsh_net_export(void* hp, int* leaf_rank, int* leaf_labels, double* leaf_data, int* output_labels,
                     int* open_labels, int* open_qubits) {
    const Handle* h = static_cast<Handle*>(hp);
    std::size_t li = 0, di = 0;
    for (std::size_t t = 0; t < h->net.tensors.size(); ++t) {
        const Tensor& tt = h->net.tensors[t];
        leaf_rank[t] = tt.rank();
        for (Label l : tt.labels) leaf_labels[li++] = l;
        for (const cplx& v : tt.data) {
            leaf_data[2 * di] = v.real();
            leaf_data[2 * di + 1] = v.imag();
            ++di;
        }
    }
    for (int q = 0; q < h->net.n_qubits; ++q) output_labels[q] = h->net.output_labels[q];
    for (std::size_t i = 0; i < h->net.open_labels.size(); ++i) {
        open_labels[i] = h->net.open_labels[i];
        open_qubits[i] = h->net.open_qubits[i];
    }
}

std::int64_t rcsh_label_names(void* hp, char* buf, std::int64_t cap) {
    const Handle* h = static_cast<Handle*>(hp);
    std::string s;
    for (const auto& n : h->net.label_names) s += n + "\n";
    if (buf && cap >= static_cast<std::int64_t>(s.size())) std::memcpy(buf, s.data(), s.size());
    return static_cast<std::int64_t>(s.size());
}

void rcsh_wire_edges(void* hp, int* out) {
    const Handle* h = static_cast<Handle*>(hp);
    for (std::size_t i = 0; i < h->net.wire_edges.size(); ++i) {
        out[3 * i] = h->net.wire_edges[i].label;
        out[3 * i + 1] = h->net.wire_edges[i].qubit;
        out[3 * i + 2] = h->net.wire_edges[i].layer;
    }
}

void rcsh_plan_sizes(void* hp, std::int64_t* sizes) {
    const Handle* h = static_cast<Handle*>(hp);
    sizes[0] = static_cast<std::int64_t>(h->plan.steps.size());
    sizes[1] = static_cast<std::int64_t>(h->plan.sliced.size());
    sizes[2] = static_cast<std::int64_t>(h->plan.broken.size());
    sizes[3] = static_cast<std::int64_t>(h->plan.fixed_outputs.size());
    sizes[4] = h->has_config ? static_cast<std::int64_t>(h->config.configurations.size()) : 0;
}

void rcsh_plan_export(void* hp, std::int64_t* steps, int* sliced, int* broken, int* fixed,
                      std::uint64_t* configs, std::uint64_t* totals) {
    const Handle* h = static_cast<Handle*>(hp);
    for (std::size_t s = 0; s < h->plan.steps.size(); ++s) {
        const PlanStep& st = h->plan.steps[s];
        steps[6 * s] = st.lhs;
        steps[6 * s + 1] = st.rhs;
        steps[6 * s + 2] = st.result;
        steps[6 * s + 3] = static_cast<std::int64_t>(st.summed);
        steps[6 * s + 4] = static_cast<std::int64_t>(st.flops);
        steps[6 * s + 5] = static_cast<std::int64_t>(st.result_bytes);
    }
    for (std::size_t i = 0; i < h->plan.sliced.size(); ++i) sliced[i] = h->plan.sliced[i];
    for (std::size_t i = 0; i < h->plan.broken.size(); ++i) broken[i] = h->plan.broken[i];
    for (std::size_t i = 0; i < h->plan.fixed_outputs.size(); ++i) fixed[i] = h->plan.fixed_outputs[i];
    if (h->has_config)
        for (std::size_t i = 0; i < h->config.configurations.size(); ++i) configs[i] = h->config.configurations[i];
    totals[0] = h->plan.flops_per_slice;
    totals[1] = h->plan.traffic_bytes_per_slice;
    totals[2] = h->plan.peak_bytes;
    totals[3] = h->plan.memory_budget_bytes;
}

std::int64_t rcsh_circuit_gates(void* hp, int* out) {
    const Handle* h = static_cast<Handle*>(hp);
    std::int64_t n = 0;
    for (std::size_t t = 0; t < h->circuit.layers.size(); ++t)
        for (const Gate& g : h->circuit.layers[t].gates) {
            if (out) {
                out[4 * n] = static_cast<int>(t);
                out[4 * n + 1] = static_cast<int>(g.kind);
                out[4 * n + 2] = g.targets[0];
                out[4 * n + 3] = g.targets.size() > 1 ? g.targets[1] : -1;
            }
            ++n;
        }
    return n;
}

// simulate_exact (statevector.cpp:79-86) of the handle's circuit into a DEVICE
// buffer of 2^n interleaved complex f64 (rcsg_statevector).
int rcsh_statevector(void* hp, double* d_state) {
    return guarded([&] {
        const Handle* h = static_cast<Handle*>(hp);
        std::vector<std::int32_t> nt, tg;
        std::vector<double> u;
        for (const Layer& layer : h->circuit.layers)
            for (const Gate& g : layer.gates) {
                nt.push_back(static_cast<std::int32_t>(g.targets.size()));
                tg.push_back(g.targets[0]);
                tg.push_back(g.targets.size() > 1 ? g.targets[1] : -1);
                for (int r = 0; r < 16; ++r) {
                    const cplx v = r < static_cast<int>(g.unitary.size()) ? g.unitary[r] : cplx(0.0, 0.0);
                    u.push_back(v.real());
                    u.push_back(v.imag());
                }
            }
        if (int rc = rcsg_statevector(h->circuit.n_qubits, static_cast<std::int32_t>(nt.size()), nt.data(),
                                      tg.data(), u.data(), d_state))
            raise_rcsg(rc);
    });
}

// rcsg_contract_groups over the handle's plan; n_cfg < 0 uses the handle's
// BrokenEdgeConfig (all m configurations), n_cfg == 0 the exact contraction.
int rcsh_contract_groups(void* hp, int precision, std::uint64_t budget, std::uint64_t n_groups,
                         const std::uint64_t* fixed, int n_cfg, const std::uint64_t* cfgs, std::uint64_t s0,
                         std::uint64_t s1, double* out, rcsg_stats* st) {
    return guarded([&] {
        Handle* h = static_cast<Handle*>(hp);
        rcsg_program* p = h->program(precision, budget);
        const std::uint64_t* c = cfgs;
        std::uint64_t nc = static_cast<std::uint64_t>(std::max(n_cfg, 0));
        if (n_cfg < 0) {
            c = h->config.configurations.data();
            nc = h->has_config ? h->config.configurations.size() : 0;
        }
        if (int rc = rcsg_contract_groups(p, n_groups, fixed, nc, c, s0, s1, out, st)) raise_rcsg(rc);
    });
}

int rcsh_contract_groups_device(void* hp, int precision, std::uint64_t budget, std::uint64_t n_groups,
                                const std::uint64_t* fixed, int n_cfg, const std::uint64_t* cfgs,
                                std::uint64_t s0, std::uint64_t s1, double* d_acc, rcsg_stats* st, int sync) {
    return guarded([&] {
        Handle* h = static_cast<Handle*>(hp);
        rcsg_program* p = h->program(precision, budget);
        const std::uint64_t* c = cfgs;
        std::uint64_t nc = static_cast<std::uint64_t>(std::max(n_cfg, 0));
        if (n_cfg < 0) {
            c = h->config.configurations.data();
            nc = h->has_config ? h->config.configurations.size() : 0;
        }
        if (int rc = rcsg_contract_groups_device(p, n_groups, fixed, nc, c, s0, s1, d_acc, sync, st)) raise_rcsg(rc);
    });
}

// wait for a program's stream and report a deferred NumericFault
int rcsh_program_sync(void* hp, int precision, std::uint64_t budget) {
    return guarded([&] {
        Handle* h = static_cast<Handle*>(hp);
        if (int rc = rcsg_program_sync(h->program(precision, budget))) raise_rcsg(rc);
    });
}

// rcs::contract with explicit fixed outputs; n_cfg < 0: handle's config, 0: exact.
int rcsh_contract(void* hp, int precision, int n_fixed, const int* labels, const int* values, int n_cfg,
                  const std::uint64_t* cfgs, double* out, std::uint64_t* flops) {
    return guarded([&] {
        Handle* h = static_cast<Handle*>(hp);
        set_precision(precision == 0 ? "f64" : precision == 1 ? "f32" : precision == 2 ? "tf32" : precision == 3 ? "3xtf32" : precision == 4 ? "bf16" : "f16");
        std::map<Label, int> fixed;
        for (int i = 0; i < n_fixed; ++i) fixed[labels[i]] = values[i];
        BrokenEdgeConfig cfg = h->config;
        if (n_cfg > 0) cfg.configurations.assign(cfgs, cfgs + n_cfg);
        const bool use = h->has_config && n_cfg != 0;
        ContractResult r = contract(h->net, h->plan, use ? &cfg : nullptr, fixed, 1);
        copy_amps(r.amplitudes, out);
        if (flops) *flops = r.stats.flops;
    });
}

// rcs::execute_assignment; call with out == nullptr first to size the result.
int rcsh_execute(void* hp, int precision, int n, const int* labels, const int* values, double* out,
                 std::int64_t* n_out) {
    return guarded([&] {
        Handle* h = static_cast<Handle*>(hp);
        set_precision(precision == 0 ? "f64" : precision == 1 ? "f32" : precision == 2 ? "tf32" : precision == 3 ? "3xtf32" : precision == 4 ? "bf16" : "f16");
        std::map<Label, int> a;
        for (int i = 0; i < n; ++i) a[labels[i]] = values[i];
        std::vector<cplx> v = execute_assignment(h->net, h->plan, a);
        if (out) copy_amps(v, out);
        *n_out = static_cast<std::int64_t>(v.size());
    });
}

int rcsh_candidates(int n, const int* open, int l, std::uint64_t n_groups, std::uint64_t seed,
                    std::uint64_t* out_fixed, int* dup) {
    return guarded([&] {
        CandidateSet cs = build_candidate_set(n, std::vector<int>(open, open + l), n_groups, seed);
        for (std::size_t g = 0; g < cs.group_fixed.size(); ++g) out_fixed[g] = cs.group_fixed[g];
        if (dup) *dup = cs.duplicate_groups;
    });
}

// rcs::top_k_select / direct_sample with probs [n_groups][2^l] as the ProbFn.
// state_fidelity (contraction_engine.cpp:327-345) over interleaved complex
// arrays; *warn = 1 for the zero-norm-approximation warning
int rcsh_state_fidelity(std::uint64_t n, const double* approx, const double* exact, double* out, int* warn) {
    return guarded([&] {
        std::vector<cplx> a(n), e(n);
        for (std::uint64_t i = 0; i < n; ++i) {
            a[i] = cplx(approx[2 * i], approx[2 * i + 1]);
            e[i] = cplx(exact[2 * i], exact[2 * i + 1]);
        }
        const FidelityResult r = state_fidelity(a, e);
        *out = r.value;
        if (warn) *warn = r.zero_norm_warning ? 1 : 0;
    });
}

// predicted_topk_xeb (sampling.cpp:147-151)
int rcsh_predicted_topk_xeb(double fidelity, std::uint64_t candidate_size, std::uint64_t k, double* out) {
    return guarded([&] { *out = predicted_topk_xeb(fidelity, candidate_size, k); });
}

// ---- artifact formats (artifacts.cpp) ----------------------------------------
namespace {
std::int64_t copy_out(const std::string& s, char* buf, std::int64_t cap) {
    if (buf && cap > 0) {
        const std::size_t m = std::min<std::size_t>(s.size(), static_cast<std::size_t>(cap - 1));
        std::memcpy(buf, s.data(), m);
        buf[m] = 0;
    }
    return static_cast<std::int64_t>(s.size());
}
}  // namespace

// plan_to_json of the handle's plan (returns its length; buf may be null)
std::int64_t rcsh_plan_json(void* hp, char* buf, std::int64_t cap) {
    const Handle* h = static_cast<Handle*>(hp);
    return copy_out(plan_to_json(h->plan, h->net), buf, cap);
}

// plan_from_json: replace the handle's plan (its compiled programs are dropped)
int rcsh_plan_import(void* hp, const char* json) {
    return guarded([&] {
        Handle* h = static_cast<Handle*>(hp);
        ContractionPlan plan = plan_from_json(json, h->net);
        for (auto& [k, p] : h->programs) rcsg_program_free(p);
        h->programs.clear();
        h->flat.reset();
        h->plan = std::move(plan);
        if (h->has_config && h->config.broken_labels != h->plan.broken) h->has_config = false;
    });
}

std::int64_t rcsh_timings_csv(int n, const std::uint64_t* ids, const std::uint64_t* bits, const double* ms,
                              const std::uint64_t* flops, char* buf, std::int64_t cap) {
    std::vector<SubtaskTiming> t(n);
    for (int i = 0; i < n; ++i) t[i] = SubtaskTiming{ids[i], bits[i], ms[i], flops[i]};
    return copy_out(timings_to_csv(t), buf, cap);
}

std::int64_t rcsh_samples_text(int n_qubits, int topk, std::uint64_t k, std::int64_t count,
                               const std::uint64_t* samples, char* buf, std::int64_t cap) {
    SampleSet ss;
    ss.n_qubits = n_qubits;
    ss.provenance = topk ? Provenance::TopK : Provenance::Direct;
    ss.k = k;
    ss.bitstrings.assign(samples, samples + count);
    return copy_out(samples_to_text(ss), buf, cap);
}

// samples_from_text: header into meta = {n_qubits, topk, k}; returns the sample
// count (out may be null to size the buffer)
std::int64_t rcsh_samples_parse(const char* text, std::uint64_t* meta, std::uint64_t* out) {
    const SampleSet ss = samples_from_text(text);
    if (meta) {
        meta[0] = static_cast<std::uint64_t>(ss.n_qubits);
        meta[1] = ss.provenance == Provenance::TopK ? 1 : 0;
        meta[2] = ss.k;
    }
    if (out) std::copy(ss.bitstrings.begin(), ss.bitstrings.end(), out);
    return static_cast<std::int64_t>(ss.bitstrings.size());
}

int rcsh_topk(int n, const int* open, int l, std::uint64_t n_groups, const std::uint64_t* fixed,
              const double* probs, std::uint64_t k, std::uint64_t* out) {
    return guarded([&] {
        CandidateSet cs = make_set(n, open, l, n_groups, fixed);
        SampleSet s = top_k_select(cs, prob_map(cs, probs), k);
        std::copy(s.bitstrings.begin(), s.bitstrings.end(), out);
    });
}

int rcsh_direct(int n, const int* open, int l, std::uint64_t n_groups, const std::uint64_t* fixed,
                const double* probs, std::uint64_t seed, std::uint64_t* out) {
    return guarded([&] {
        CandidateSet cs = make_set(n, open, l, n_groups, fixed);
        SampleSet s = direct_sample(cs, prob_map(cs, probs), seed);
        std::copy(s.bitstrings.begin(), s.bitstrings.end(), out);
    });
}

std::uint64_t rcsh_member(int n, const int* open, int l, std::uint64_t fixed, std::uint64_t i) {
    CandidateSet cs = make_set(n, open, l, 1, &fixed);
    return cs.member(0, i);
}

std::uint64_t rcsh_rng_split_next(std::uint64_t seed, std::uint64_t tag) {
    return Rng(seed).split(tag).next_u64();
}

std::uint64_t rcsh_lexkey(std::uint64_t index, int n) { return lexicographic_key(index, n); }

int rcsh_broken_configs(int k, std::uint64_t m, std::uint64_t seed, std::uint64_t* out) {
    return guarded([&] {
        BrokenEdgeConfig c = make_broken_config(std::vector<Label>(k, 0), m, seed);
        std::copy(c.configurations.begin(), c.configurations.end(), out);
    });
}

}  // extern "C"
