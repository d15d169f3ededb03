// Host C++ API (namespace rcs) of the hot path, implemented over the C ABI.
//
// Same signatures, validation, error types and result semantics as the
// reference executor (contraction_engine.cpp:132-354); every contraction runs
// on the GPU (rcsg.h) — there is no CPU execution path.
#include <chrono>
#include <istream>
#include <ostream>
#include <cmath>
#include <cstring>
#include <algorithm>
#include <memory>
#include <mutex>

#include "rcs_b200.hpp"
#include "flat.hpp"
#include "rcsg.h"

namespace rcs {
namespace {

int g_precision = RCSG_PREC_F64;

[[noreturn]] void raise(int rc) {
    int32_t step = -1;
    const std::string msg = rcsg_last_error(&step);
    switch (rc) {
        case RCSG_ERR_CONFIG: throw ConfigError(msg);
        case RCSG_ERR_NUMERIC: throw NumericFault(msg, step);
        case RCSG_ERR_CAPACITY: throw CapacityError(msg);
        default: throw DeviceError(msg);
    }
}
void ok(int rc) {
    if (rc) raise(rc);
}

// ---- compiled-program cache --------------------------------------------------
// The reference re-interprets the plan on every call; compiling a device
// program (layouts, reassociation, fp16 calibration, binding, graph capture)
// is the expensive part here, so programs are cached by a fingerprint of the
// flattened (network, plan), the precision and the pins, LRU over kCacheSize
// entries.  Calls are serialised by the cache lock (a program is not
// re-entrant, and one host thread drives the device anyway).
constexpr std::size_t kCacheSize = 8;

std::uint64_t fnv(std::uint64_t h, const void* p, std::size_t n) {
    const auto* b = static_cast<const unsigned char*>(p);
    for (std::size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 0x100000001b3ull;
    return h;
}
template <class V>
std::uint64_t fnv_vec(std::uint64_t h, const V& v) {
    const std::uint64_t n = v.size();
    h = fnv(h, &n, sizeof n);
    return v.empty() ? h : fnv(h, v.data(), v.size() * sizeof(v[0]));
}
std::uint64_t fingerprint(const Flat& f) {
    std::uint64_t h = 0xcbf29ce484222325ull;
    for (const auto* v : {&f.rank, &f.labels, &f.out_l, &f.open_l, &f.open_q, &f.steps, &f.sliced, &f.broken, &f.fixed})
        h = fnv_vec(h, *v);
    return fnv_vec(h, f.data);
}

struct Cached {
    std::uint64_t key = 0;
    int precision = 0;
    int kind = 0;  // 0 group program, 1 pinned program, 2 multi-device program
    std::vector<int8_t> pins;
    rcsg_program* prog = nullptr;
    rcsg_multi* multi = nullptr;
    std::uint64_t used = 0;
};

std::mutex g_mu;  // guards the cache, the device context and every device call below
std::vector<Cached> g_cache;
std::uint64_t g_tick = 0;
rcsg_context* g_ctx = nullptr;
int g_ctx_devices = 0;

void free_entry(Cached& c) {
    if (c.prog) rcsg_program_free(c.prog);
    if (c.multi) rcsg_multi_free(c.multi);
    c.prog = nullptr;
    c.multi = nullptr;
}

Cached& cached(const Flat& f, int kind, const std::vector<int8_t>& pins) {
    const std::uint64_t key = fingerprint(f);
    for (Cached& c : g_cache)
        if (c.key == key && c.kind == kind && c.precision == g_precision && c.pins == pins) {
            c.used = ++g_tick;
            return c;
        }
    if (g_cache.size() >= kCacheSize) {
        auto lru = std::min_element(g_cache.begin(), g_cache.end(),
                                    [](const Cached& a, const Cached& b) { return a.used < b.used; });
        free_entry(*lru);
        g_cache.erase(lru);
    }
    Cached c;
    c.key = key;
    c.kind = kind;
    c.precision = g_precision;
    c.pins = pins;
    c.used = ++g_tick;
    if (kind == 0) ok(rcsg_compile(&f.net, &f.plan, g_precision, 0, &c.prog));
    else if (kind == 1) ok(rcsg_compile_pinned(&f.net, &f.plan, g_precision, 0, pins.data(), &c.prog));
    else ok(rcsg_context_compile(g_ctx, &f.net, &f.plan, g_precision, 0, 0, &c.multi));
    g_cache.push_back(std::move(c));
    return g_cache.back();
}

// group code of a fixed_outputs map that pins exactly the non-open output legs
// (contract_group's packing, contraction_engine.cpp:310-318); false otherwise
bool as_group(const TensorNetwork& network, const std::map<Label, int>& fixed, std::uint64_t& code) {
    code = 0;
    std::size_t n_fixed = 0;
    int bit = 0;
    for (int q = 0; q < network.n_qubits; ++q) {
        if (std::find(network.open_qubits.begin(), network.open_qubits.end(), q) != network.open_qubits.end()) continue;
        auto it = fixed.find(network.output_labels[q]);
        if (it == fixed.end()) return false;
        if (it->second) code |= std::uint64_t{1} << bit;
        ++bit;
        ++n_fixed;
    }
    return n_fixed == fixed.size() && bit <= 64;
}

void check_config(const ContractionPlan& plan, const BrokenEdgeConfig* config) {
    if (config) {
        if (config->broken_labels != plan.broken)
            throw ConfigError("broken-edge labels do not match the plan");
        if (config->configurations.empty()) throw ConfigError("broken-edge configuration list is empty");
    } else if (!plan.broken.empty()) {
        throw ConfigError("plan has broken edges; exact contraction needs a plan without them");
    }
}

std::vector<cplx> to_cplx(const std::vector<double>& v) {
    std::vector<cplx> out(v.size() / 2);
    for (std::size_t i = 0; i < out.size(); ++i) out[i] = cplx(v[2 * i], v[2 * i + 1]);
    return out;
}

}  // namespace

void set_precision(const std::string& p) {
    if (p == "f64") g_precision = RCSG_PREC_F64;
    else if (p == "f32") g_precision = RCSG_PREC_F32;
    else if (p == "tf32") g_precision = RCSG_PREC_TF32;
    else if (p == "3xtf32") g_precision = RCSG_PREC_3XTF32;
    else if (p == "bf16") g_precision = RCSG_PREC_BF16;
    else if (p == "f16") g_precision = RCSG_PREC_F16;
    else throw ConfigError("precision must be f64, f32, tf32, 3xtf32, bf16 or f16");
}

std::string get_precision() {
    static const char* names[] = {"f64", "f32", "tf32", "3xtf32", "bf16", "f16"};
    return names[g_precision];
}

double BrokenEdgeConfig::predicted_fidelity() const {
    return static_cast<double>(m()) * std::pow(2.0, -k());
}

BrokenEdgeConfig make_broken_config(std::vector<Label> broken_labels, std::uint64_t m, std::uint64_t seed) {
    const int k = static_cast<int>(broken_labels.size());
    if (k > 62) throw ConfigError("too many broken edges");
    const std::uint64_t full = std::uint64_t{1} << k;
    if (m < 1 || m > full)
        throw ConfigError("configuration count m=" + std::to_string(m) + " outside [1, 2^" +
                          std::to_string(k) + "]");
    BrokenEdgeConfig c;
    c.broken_labels = std::move(broken_labels);
    // Gray-code walk from a seeded start (contraction_engine.cpp:136-151)
    const std::uint64_t start = Rng(seed ^ 0xb20ced6eULL).next_below(full);
    for (std::uint64_t i = 0; i < m; ++i) c.configurations.push_back(start ^ i ^ (i >> 1));
    return c;
}

std::vector<cplx> execute_assignment(const TensorNetwork& network, const ContractionPlan& plan,
                                     const std::map<Label, int>& assignment, ExecutionStats* stats) {
    const int n_labels = static_cast<int>(network.label_names.size());
    std::vector<int8_t> pin(n_labels, -1);
    for (const auto& [l, v] : assignment) {
        if (l < 0 || l >= n_labels) throw ConfigError("assignment label " + std::to_string(l) + " not in network");
        if (v != 0 && v != 1) throw ConfigError("assignment values must be 0/1");
        pin[l] = static_cast<int8_t>(v);
    }
    auto f = flatten(network, plan);
    uint64_t n = 0;
    ok(rcsg_execute_assignment(&f->net, &f->plan, g_precision, pin.data(), nullptr, &n));
    std::vector<double> out(2 * n);
    ok(rcsg_execute_assignment(&f->net, &f->plan, g_precision, pin.data(), out.data(), &n));
    if (stats) stats->flops += plan.flops_per_slice;
    return to_cplx(out);
}

ContractResult contract(const TensorNetwork& network, const ContractionPlan& plan,
                        const BrokenEdgeConfig* config, const std::map<Label, int>& fixed_outputs,
                        int workers) {
    if (workers < 1) throw ConfigError("workers must be >= 1");
    check_config(plan, config);
    const int n_labels = static_cast<int>(network.label_names.size());
    std::vector<int8_t> pin(n_labels, -1);
    for (const auto& [l, v] : fixed_outputs) {
        if (l < 0 || l >= n_labels) throw ConfigError("assignment label " + std::to_string(l) + " not in network");
        if (v != 0 && v != 1) throw ConfigError("assignment values must be 0/1");
        pin[l] = static_cast<int8_t>(v);
    }
    auto f = flatten(network, plan);
    std::lock_guard<std::mutex> lock(g_mu);
    // with a device context, a group-shaped pin set runs sharded over
    // min(workers, devices) GPUs (canonical slice blocks: results do not depend
    // on `workers`, like the reference's thread pool, contraction_engine.cpp:264-287)
    std::uint64_t code = 0;
    const bool multi = g_ctx && as_group(network, fixed_outputs, code);
    Cached& c = multi ? cached(*f, 2, {}) : cached(*f, 1, pin);
    const std::vector<std::uint64_t> none{0};
    const std::vector<std::uint64_t>& cfgs = config ? config->configurations : none;
    ContractResult res;
    std::vector<double> sum, comp;
    const std::uint64_t group = multi ? code : 0;
    std::size_t n = std::size_t{1} << network.open_labels.size();
    if (!multi)
        for (Label l : network.open_labels)
            if (pin[l] >= 0) n >>= 1;
    for (std::size_t t = 0; t < cfgs.size(); ++t) {
        rcsg_stats st{};
        const auto t0 = std::chrono::steady_clock::now();
        // one subtask = one configuration over every slice (contraction_engine.cpp:237-262)
        std::vector<double> buf(2 * n, 0.0);
        if (multi)
            ok(rcsg_multi_contract_groups(c.multi, 1, &group, config ? 1 : 0, config ? &cfgs[t] : nullptr, 0,
                                          plan.n_slices(), workers, buf.data(), &st));
        else
            ok(rcsg_contract_groups(c.prog, 1, &group, config ? 1 : 0, config ? &cfgs[t] : nullptr, 0,
                                    plan.n_slices(), buf.data(), &st));
        const auto t1 = std::chrono::steady_clock::now();
        if (sum.empty()) {
            sum.assign(buf.size(), 0.0);
            comp.assign(buf.size(), 0.0);
        }
        // compensated reduction in ascending configuration order (:289-302)
        for (std::size_t i = 0; i < buf.size(); ++i) {
            const double y = buf[i] - comp[i];
            const double s = sum[i] + y;
            comp[i] = (s - sum[i]) - y;
            sum[i] = s;
        }
        res.timings.push_back({t, cfgs[t], std::chrono::duration<double, std::milli>(t1 - t0).count(),
                               plan.flops_per_slice * plan.n_slices()});
        res.stats.flops += plan.flops_per_slice * plan.n_slices();
        res.stats.peak_bytes = std::max<std::uint64_t>(res.stats.peak_bytes, st.arena_bytes);
    }
    res.amplitudes = to_cplx(sum);
    return res;
}

AmplitudeBatch contract_group(const TensorNetwork& network, const ContractionPlan& plan,
                              const BrokenEdgeConfig* config, std::uint64_t group_id,
                              std::uint64_t fixed_bits) {
    auto all = contract_groups(network, plan, config, {fixed_bits});
    AmplitudeBatch b = std::move(all[0]);
    b.group_id = group_id;
    return b;
}

std::vector<AmplitudeBatch> contract_groups(const TensorNetwork& network, const ContractionPlan& plan,
                                            const BrokenEdgeConfig* config,
                                            const std::vector<std::uint64_t>& group_fixed) {
    check_config(plan, config);
    if (group_fixed.empty()) throw ConfigError("group count must be >= 1");
    auto f = flatten(network, plan);
    std::lock_guard<std::mutex> lock(g_mu);
    Cached& c = cached(*f, 0, {});
    const int l = static_cast<int>(network.open_labels.size());
    const std::size_t per = std::size_t{1} << l;
    std::vector<double> out(2 * per * group_fixed.size());
    const std::size_t n_cfg = config ? config->configurations.size() : 0;
    ok(rcsg_contract_groups(c.prog, group_fixed.size(), group_fixed.data(), n_cfg,
                            config ? config->configurations.data() : nullptr, 0, plan.n_slices(), out.data(),
                            nullptr));
    std::vector<AmplitudeBatch> res(group_fixed.size());
    for (std::size_t g = 0; g < group_fixed.size(); ++g) {
        res[g].group_id = g;
        res[g].n_open = l;
        res[g].fixed_bits = group_fixed[g];
        res[g].amplitudes.resize(per);
        for (std::size_t i = 0; i < per; ++i)
            res[g].amplitudes[i] = cplx(out[2 * (g * per + i)], out[2 * (g * per + i) + 1]);
    }
    return res;
}

void init_devices(const std::vector<int>& devices) {
    std::lock_guard<std::mutex> lock(g_mu);
    for (Cached& c : g_cache) free_entry(c);
    g_cache.clear();
    if (g_ctx) rcsg_context_free(g_ctx);
    g_ctx = nullptr;
    g_ctx_devices = 0;
    if (devices.empty()) return;
    std::vector<std::int32_t> d(devices.begin(), devices.end());
    ok(rcsg_init(d.data(), static_cast<std::int32_t>(d.size()), &g_ctx));
    g_ctx_devices = static_cast<int>(d.size());
}

int device_count() {
    std::lock_guard<std::mutex> lock(g_mu);
    return g_ctx_devices;
}

void clear_program_cache() {
    std::lock_guard<std::mutex> lock(g_mu);
    for (Cached& c : g_cache) free_entry(c);
    g_cache.clear();
}

FidelityResult state_fidelity(std::span<const cplx> approx, std::span<const cplx> exact) {
    if (approx.size() != exact.size()) throw ConfigError("fidelity requires identical index sets");
    cplx overlap(0.0, 0.0);
    double na = 0.0, ne = 0.0;
    for (std::size_t i = 0; i < approx.size(); ++i) {
        overlap += std::conj(exact[i]) * approx[i];
        na += std::norm(approx[i]);
        ne += std::norm(exact[i]);
    }
    if (ne == 0.0) throw ConfigError("exact collection has zero norm");
    FidelityResult r;
    if (na == 0.0) {
        r.zero_norm_warning = true;
        return r;
    }
    r.value = std::norm(overlap) / (na * ne);
    return r;
}

}  // namespace rcs

// ---- exact statevector (statevector.cpp), computed by rcsg_statevector ------
namespace rcs {

double StateVector::norm_sq() const {
    double s = 0.0;
    for (const cplx& a : amps) s += std::norm(a);
    return s;
}

StateVector simulate_exact(const Circuit& circuit, int cap) {
    if (circuit.n_qubits > cap)
        throw CapacityError("exact simulation capped at " + std::to_string(cap) + " qubits, circuit has " +
                            std::to_string(circuit.n_qubits));
    std::vector<std::int32_t> nt, tg;
    std::vector<double> u;
    for (const Layer& layer : circuit.layers)
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
    StateVector st;
    st.n_qubits = circuit.n_qubits;
    const std::size_t dim = std::size_t{1} << circuit.n_qubits;
    void* d = nullptr;
    ok(rcsg_device_alloc(dim * 2 * sizeof(double), &d));
    std::unique_ptr<void, void (*)(void*)> hold(d, [](void* p) { rcsg_device_free(p); });
    ok(rcsg_statevector(circuit.n_qubits, static_cast<std::int32_t>(nt.size()), nt.data(), tg.data(), u.data(),
                        static_cast<double*>(d)));
    st.amps.resize(dim);
    ok(rcsg_memcpy(st.amps.data(), d, dim * 2 * sizeof(double), 2));
    return st;
}

std::uint64_t bitstring_to_index(const std::string& bitstring) {
    std::uint64_t idx = 0;
    for (std::size_t q = 0; q < bitstring.size(); ++q) {
        const char c = bitstring[q];
        if (c != '0' && c != '1') throw ConfigError("bitstring must be 0/1");
        if (c == '1') idx |= std::uint64_t{1} << q;
    }
    return idx;
}

std::string index_to_bitstring(std::uint64_t index, int n_qubits) {
    std::string s(n_qubits, '0');
    for (int q = 0; q < n_qubits; ++q)
        if ((index >> q) & 1) s[q] = '1';
    return s;
}

void dump_amplitudes(const StateVector& state, std::ostream& out) {
    char header[16] = {0};
    const std::uint32_t version = 1, n = static_cast<std::uint32_t>(state.n_qubits);
    std::memcpy(header, "QSVD", 4);
    std::memcpy(header + 4, &version, 4);
    std::memcpy(header + 8, &n, 4);
    out.write(header, 16);
    // std::complex<double> is two contiguous doubles (re, im): one bulk write
    out.write(reinterpret_cast<const char*>(state.amps.data()),
              static_cast<std::streamsize>(state.amps.size() * sizeof(cplx)));
}

StateVector load_amplitudes(std::istream& in) {
    char header[16];
    in.read(header, 16);
    if (!in || std::memcmp(header, "QSVD", 4) != 0) throw ConfigError("bad amplitude dump header");
    std::uint32_t n = 0;
    std::memcpy(&n, header + 8, 4);
    if (n > 40) throw ConfigError("bad amplitude dump header");
    StateVector st;
    st.n_qubits = static_cast<int>(n);
    st.amps.resize(std::size_t{1} << n);
    in.read(reinterpret_cast<char*>(st.amps.data()), static_cast<std::streamsize>(st.amps.size() * sizeof(cplx)));
    if (!in) throw ConfigError("truncated amplitude dump");
    return st;
}

double ideal_probability(const StateVector& state, const std::string& bitstring) {
    if (static_cast<int>(bitstring.size()) != state.n_qubits) throw ConfigError("bitstring length mismatch");
    return std::norm(state.amps[bitstring_to_index(bitstring)]);
}

}  // namespace rcs
