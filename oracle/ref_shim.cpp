// TEST INFRASTRUCTURE ONLY — flat C ABI over the UNMODIFIED reference library
// (/root/reference/proj, compiled by oracle/Makefile into oracle/_ref/).
//
// Used by: tests/ (parity against the reference itself), tests/golden/make_golden.py
// (fixture generation), and bench.py's `cpu_baseline` / `--impl reference` legs.
// Never linked into, or called by, the product library.
//
// Each entry point wraps one public reference call:
//   refo_build           gen_random_circuit (circuit.cpp:112), circuit_to_network
//                        (tensor_network.cpp:20), select_broken_edges
//                        (contraction_plan.cpp:379), find_contraction_path (:308),
//                        make_broken_config (contraction_engine.cpp:136)
//   refo_contract        contract (contraction_engine.cpp:210)
//   refo_contract_group  contract_group (contraction_engine.cpp:307)
//   refo_execute         execute_assignment (contraction_engine.cpp:153)
//   refo_exact           simulate_exact (statevector.cpp:79)
//   refo_candidates      build_candidate_set (sampling.cpp:29)
//   refo_topk            top_k_select (sampling.cpp:82)
//   refo_direct          direct_sample (sampling.cpp:116)
//   refo_xeb             xeb (sampling.cpp:62)
//   refo_plan_json       plan_to_json (contraction_plan.cpp:451)
//   refo_set_plan        replaces the handle's plan steps / sliced labels (plans
//                        imported from the product's scale planner run on the
//                        reference executor)
//   refo_timings_csv     contract + timings_to_csv (contraction_engine.cpp:347)
//   refo_samples_text    samples_to_text / samples_from_text (sampling.cpp:177-210)
#include <chrono>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "rcs/circuit.hpp"
#include "rcs/contraction_engine.hpp"
#include "rcs/contraction_plan.hpp"
#include "rcs/errors.hpp"
#include "rcs/rng.hpp"
#include "rcs/sampling.hpp"
#include "rcs/statevector.hpp"
#include "rcs/tensor_network.hpp"

using namespace rcs;

namespace {

thread_local std::string g_err;
thread_local int g_err_step = -1;

struct Handle {
    Circuit circuit;
    TensorNetwork net;
    ContractionPlan plan;
    BrokenEdgeConfig config;
    bool has_config = false;
};

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const NumericFault& e) {
        g_err = e.what();
        g_err_step = e.step_index;
        return e.exit_code;
    } catch (const Error& e) {
        g_err = e.what();
        return e.exit_code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

SearchEffort effort_of(int e) {
    return e == 0 ? SearchEffort::Low : (e == 2 ? SearchEffort::High : SearchEffort::Medium);
}

void copy_amps(const std::vector<cplx>& v, double* out) {
    for (std::size_t i = 0; i < v.size(); ++i) {
        out[2 * i] = v[i].real();
        out[2 * i + 1] = v[i].imag();
    }
}

ProbFn prob_map(int n_groups, int l, const CandidateSet& cs, const double* probs) {
    auto map = std::make_shared<std::unordered_map<std::uint64_t, double>>();
    const std::uint64_t per = std::uint64_t{1} << l;
    for (int g = 0; g < n_groups; ++g)
        for (std::uint64_t i = 0; i < per; ++i) (*map)[cs.member(g, i)] = probs[g * per + i];
    return [map](std::uint64_t idx) {
        auto it = map->find(idx);
        return it == map->end() ? -1.0 : it->second;
    };
}

CandidateSet make_set(int n, const int* open, int l, int n_groups, const std::uint64_t* fixed) {
    CandidateSet cs;
    cs.n_qubits = n;
    cs.open_qubits.assign(open, open + l);
    cs.group_fixed.assign(fixed, fixed + n_groups);
    return cs;
}

}  // namespace

extern "C" {

const char* refo_last_error(int* step) {
    if (step) *step = g_err_step;
    return g_err.c_str();
}

// Pipeline for the per-group path: network with `open` legs free, K broken
// edges (select_broken_edges), plan under `budget`, m Gray configurations.
// `topology` is the reference's name ("line", "ring", "grid(R,C)").
int refo_build(int n, int cycles, const char* topology, std::uint64_t seed, const int* open,
               int n_open, std::uint64_t budget, int effort, int k_broken, std::uint64_t m,
               void** out) {
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

void refo_free(void* h) { delete static_cast<Handle*>(h); }

// sizes[0..7] = n_leaves, n_labels, n_qubits, n_open, sum(rank), sum(2^rank),
//               n_layers, n_wire_edges
void refo_net_sizes(void* hp, std::int64_t* sizes) {
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

void refo_net_export(void* hp, int* leaf_rank, int* leaf_labels, double* leaf_data,
                     int* output_labels, int* open_labels, int* open_qubits) {
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

// Label names concatenated with '\n' into buf (returns needed size).
std::int64_t refo_label_names(void* hp, char* buf, std::int64_t cap) {
    const Handle* h = static_cast<Handle*>(hp);
    std::string s;
    for (const auto& n : h->net.label_names) s += n + "\n";
    if (buf && cap >= static_cast<std::int64_t>(s.size())) std::memcpy(buf, s.data(), s.size());
    return static_cast<std::int64_t>(s.size());
}

// wire edges: label, qubit, layer triples
void refo_wire_edges(void* hp, int* out) {
    const Handle* h = static_cast<Handle*>(hp);
    for (std::size_t i = 0; i < h->net.wire_edges.size(); ++i) {
        out[3 * i] = h->net.wire_edges[i].label;
        out[3 * i + 1] = h->net.wire_edges[i].qubit;
        out[3 * i + 2] = h->net.wire_edges[i].layer;
    }
}

// sizes[0..4] = n_steps, n_sliced, n_broken, n_fixed, n_configs
void refo_plan_sizes(void* hp, std::int64_t* sizes) {
    const Handle* h = static_cast<Handle*>(hp);
    sizes[0] = static_cast<std::int64_t>(h->plan.steps.size());
    sizes[1] = static_cast<std::int64_t>(h->plan.sliced.size());
    sizes[2] = static_cast<std::int64_t>(h->plan.broken.size());
    sizes[3] = static_cast<std::int64_t>(h->plan.fixed_outputs.size());
    sizes[4] = h->has_config ? static_cast<std::int64_t>(h->config.configurations.size()) : 0;
}

// steps: [n_steps][6] = lhs, rhs, result, summed, flops, result_bytes
// totals: flops_per_slice, traffic_bytes_per_slice, peak_bytes, budget
void refo_plan_export(void* hp, std::int64_t* steps, int* sliced, int* broken, int* fixed,
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
    for (std::size_t i = 0; i < h->plan.fixed_outputs.size(); ++i)
        fixed[i] = h->plan.fixed_outputs[i];
    if (h->has_config)
        for (std::size_t i = 0; i < h->config.configurations.size(); ++i)
            configs[i] = h->config.configurations[i];
    totals[0] = h->plan.flops_per_slice;
    totals[1] = h->plan.traffic_bytes_per_slice;
    totals[2] = h->plan.peak_bytes;
    totals[3] = h->plan.memory_budget_bytes;
}

// circuit gates: per gate (layer, kind, q0, q1) with q1=-1 for single-qubit.
std::int64_t refo_circuit_gates(void* hp, int* out) {
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

// contract_group over all slices and (if the plan has broken edges) all m
// configurations of the handle's BrokenEdgeConfig.
int refo_contract_group(void* hp, std::uint64_t fixed_bits, double* out) {
    return guarded([&] {
        const Handle* h = static_cast<Handle*>(hp);
        AmplitudeBatch b = contract_group(h->net, h->plan, h->has_config ? &h->config : nullptr,
                                          0, fixed_bits);
        copy_amps(b.amplitudes, out);
    });
}

// contract() with an explicit config subset (n_cfg == 0 -> handle's config or none).
int refo_contract(void* hp, int n_fixed, const int* fixed_labels, const int* fixed_values,
                  int n_cfg, const std::uint64_t* cfgs, int workers, double* out,
                  std::uint64_t* flops) {
    return guarded([&] {
        const Handle* h = static_cast<Handle*>(hp);
        std::map<Label, int> fixed;
        for (int i = 0; i < n_fixed; ++i) fixed[fixed_labels[i]] = fixed_values[i];
        BrokenEdgeConfig cfg = h->config;
        if (n_cfg > 0) cfg.configurations.assign(cfgs, cfgs + n_cfg);
        ContractResult r = contract(h->net, h->plan, h->has_config ? &cfg : nullptr, fixed,
                                    workers);
        copy_amps(r.amplitudes, out);
        if (flops) *flops = r.stats.flops;
    });
}

// execute_assignment with a label->value assignment; returns #amps in *n_out.
int refo_execute(void* hp, int n, const int* labels, const int* values, double* out,
                 std::int64_t* n_out) {
    return guarded([&] {
        const Handle* h = static_cast<Handle*>(hp);
        std::map<Label, int> a;
        for (int i = 0; i < n; ++i) a[labels[i]] = values[i];
        std::vector<cplx> v = execute_assignment(h->net, h->plan, a);
        if (out) copy_amps(v, out);
        *n_out = static_cast<std::int64_t>(v.size());
    });
}

// Assignment for (group fixed bits, slice s, config bits) exactly as
// contract()/contract_group() build it (contraction_engine.cpp:242-248,310-318).
int refo_execute_gsc(void* hp, std::uint64_t fixed_bits, std::uint64_t slice,
                     std::uint64_t config_bits, double* out) {
    return guarded([&] {
        const Handle* h = static_cast<Handle*>(hp);
        std::map<Label, int> a;
        int bit = 0;
        for (int q = 0; q < h->net.n_qubits; ++q) {
            bool is_open = false;
            for (int oq : h->net.open_qubits) is_open = is_open || oq == q;
            if (is_open) continue;
            a[h->net.output_labels[q]] = static_cast<int>((fixed_bits >> bit) & 1);
            ++bit;
        }
        for (std::size_t b = 0; b < h->plan.broken.size(); ++b)
            a[h->plan.broken[b]] = static_cast<int>((config_bits >> b) & 1);
        for (std::size_t b = 0; b < h->plan.sliced.size(); ++b)
            a[h->plan.sliced[b]] = static_cast<int>((slice >> b) & 1);
        copy_amps(execute_assignment(h->net, h->plan, a), out);
    });
}

int refo_exact(void* hp, int cap, double* out) {
    return guarded([&] {
        const Handle* h = static_cast<Handle*>(hp);
        StateVector sv = simulate_exact(h->circuit, cap);
        copy_amps(sv.amps, out);
    });
}

int refo_candidates(int n, const int* open, int l, std::uint64_t n_groups, std::uint64_t seed,
                    std::uint64_t* out_fixed, int* dup) {
    return guarded([&] {
        CandidateSet cs = build_candidate_set(n, std::vector<int>(open, open + l), n_groups, seed);
        for (std::size_t g = 0; g < cs.group_fixed.size(); ++g) out_fixed[g] = cs.group_fixed[g];
        if (dup) *dup = cs.duplicate_groups;
    });
}

std::uint64_t refo_member(int n, const int* open, int l, std::uint64_t fixed, std::uint64_t i) {
    CandidateSet cs = make_set(n, open, l, 1, &fixed);
    return cs.member(0, i);
}

// probs: [n_groups][2^l] candidate probabilities (p of member(g, i)).
int refo_topk(int n, const int* open, int l, int n_groups, const std::uint64_t* fixed,
              const double* probs, std::uint64_t k, std::uint64_t* out) {
    return guarded([&] {
        CandidateSet cs = make_set(n, open, l, n_groups, fixed);
        SampleSet s = top_k_select(cs, prob_map(n_groups, l, cs, probs), k);
        for (std::size_t i = 0; i < s.bitstrings.size(); ++i) out[i] = s.bitstrings[i];
    });
}

int refo_direct(int n, const int* open, int l, int n_groups, const std::uint64_t* fixed,
                const double* probs, std::uint64_t rng_seed, std::uint64_t* out) {
    return guarded([&] {
        CandidateSet cs = make_set(n, open, l, n_groups, fixed);
        SampleSet s = direct_sample(cs, prob_map(n_groups, l, cs, probs), rng_seed);
        for (std::size_t i = 0; i < s.bitstrings.size(); ++i) out[i] = s.bitstrings[i];
    });
}

// q: ideal probability of each sample, in sample order.
int refo_xeb(int n, const std::uint64_t* samples, int count, const double* q, double* out) {
    return guarded([&] {
        SampleSet s;
        s.n_qubits = n;
        s.bitstrings.assign(samples, samples + count);
        std::unordered_map<std::uint64_t, double> m;
        for (int i = 0; i < count; ++i) m[samples[i]] = q[i];
        *out = xeb(s, [&m](std::uint64_t x) { return m.at(x); });
    });
}

std::uint64_t refo_rng_split_next(std::uint64_t seed, std::uint64_t tag) {
    return Rng(seed).split(tag).next_u64();
}

std::uint64_t refo_lexkey(std::uint64_t index, int n) { return lexicographic_key(index, n); }

// CPU baseline: contract_group for groups [g0, g1) of `fixed`, spread over
// `threads` host threads (contract_group itself forces workers=1,
// contraction_engine.cpp:323), results [g][2^l] interleaved into out.
// Returns wall seconds in *secs.
int refo_groups_mt(void* hp, const std::uint64_t* fixed, int n_groups, int threads, double* out,
                   double* secs) {
    return guarded([&] {
        const Handle* h = static_cast<Handle*>(hp);
        const std::size_t per = std::size_t{1} << h->net.open_qubits.size();
        std::vector<std::exception_ptr> errs(threads);
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (int w = 0; w < threads; ++w)
            pool.emplace_back([&, w] {
                try {
                    for (int g = w; g < n_groups; g += threads) {
                        AmplitudeBatch b = contract_group(
                            h->net, h->plan, h->has_config ? &h->config : nullptr, g, fixed[g]);
                        copy_amps(b.amplitudes, out + 2 * per * g);
                    }
                } catch (...) {
                    errs[w] = std::current_exception();
                }
            });
        for (auto& t : pool) t.join();
        *secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
    });
}

// CPU baseline for sliced configs: execute_assignment on `count` (group,slice)
// pairs concurrently, one per thread (the reference runs slices sequentially
// inside a subtask, contraction_engine.cpp:241-255). Returns wall seconds.
int refo_slices_mt(void* hp, std::uint64_t fixed_bits, const std::uint64_t* slices, int count,
                   int threads, double* out, double* secs) {
    return guarded([&] {
        const Handle* h = static_cast<Handle*>(hp);
        const std::size_t per = std::size_t{1} << h->net.open_qubits.size();
        std::vector<int> rc(count, 0);
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (int w = 0; w < threads; ++w)
            pool.emplace_back([&, w] {
                for (int i = w; i < count; i += threads)
                    rc[i] = refo_execute_gsc(hp, fixed_bits, slices[i], 0, out + 2 * per * i);
            });
        for (auto& t : pool) t.join();
        *secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        for (int i = 0; i < count; ++i)
            if (rc[i]) throw Error("slice execution failed: " + g_err, rc[i]);
        (void)h;
    });
}

// plan_to_json of the handle's plan into buf (returns the length; buf may be null)
std::int64_t refo_plan_json(void* hp, char* buf, std::int64_t cap) {
    const Handle* h = static_cast<Handle*>(hp);
    const std::string j = plan_to_json(h->plan, h->net);
    if (buf && cap > 0) {
        const std::size_t n = std::min<std::size_t>(j.size(), static_cast<std::size_t>(cap - 1));
        std::memcpy(buf, j.data(), n);
        buf[n] = 0;
    }
    return static_cast<std::int64_t>(j.size());
}

// Replace the plan's steps ([n][3] lhs, rhs, result) and sliced labels; the
// reference executor only reads lhs / rhs / result and the sliced list.
int refo_set_plan(void* hp, int n_steps, const int* steps, int n_sliced, const int* sliced) {
    return guarded([&] {
        Handle* h = static_cast<Handle*>(hp);
        h->plan.steps.clear();
        for (int i = 0; i < n_steps; ++i) {
            PlanStep st;
            st.lhs = steps[3 * i];
            st.rhs = steps[3 * i + 1];
            st.result = steps[3 * i + 2];
            h->plan.steps.push_back(st);
        }
        h->plan.sliced.assign(sliced, sliced + n_sliced);
    });
}

// timings_to_csv of synthetic timings (ids, config bits, wall ms, flops)
std::int64_t refo_timings_csv(int n, const std::uint64_t* ids, const std::uint64_t* bits, const double* ms,
                              const std::uint64_t* flops, char* buf, std::int64_t cap) {
    std::vector<SubtaskTiming> t(n);
    for (int i = 0; i < n; ++i) t[i] = SubtaskTiming{ids[i], bits[i], ms[i], flops[i]};
    const std::string s = timings_to_csv(t);
    if (buf && cap > 0) {
        const std::size_t m = std::min<std::size_t>(s.size(), static_cast<std::size_t>(cap - 1));
        std::memcpy(buf, s.data(), m);
        buf[m] = 0;
    }
    return static_cast<std::int64_t>(s.size());
}

// samples_to_text of (n_qubits, provenance 0 direct / 1 top-k, k, samples)
std::int64_t refo_samples_text(int n_qubits, int topk, std::uint64_t k, int count, const std::uint64_t* samples,
                               char* buf, std::int64_t cap) {
    SampleSet ss;
    ss.n_qubits = n_qubits;
    ss.provenance = topk ? Provenance::TopK : Provenance::Direct;
    ss.k = k;
    ss.bitstrings.assign(samples, samples + count);
    const std::string s = samples_to_text(ss);
    if (buf && cap > 0) {
        const std::size_t m = std::min<std::size_t>(s.size(), static_cast<std::size_t>(cap - 1));
        std::memcpy(buf, s.data(), m);
        buf[m] = 0;
    }
    return static_cast<std::int64_t>(s.size());
}

}  // extern "C"
