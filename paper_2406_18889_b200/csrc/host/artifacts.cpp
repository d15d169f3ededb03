// Artifact formats of the path, byte-compatible with the
// reference's writers so files interchange in both directions:
//   plan_to_json / plan_from_json   contraction_plan.cpp:451-491 (plan.json;
//                                   import rebuilds the post-order steps from
//                                   the nested "order" and the sliced/broken names)
//   timings_to_csv                  contraction_engine.cpp:347-354 (timings.csv)
//   samples_to_text / _from_text    sampling.cpp:177-210 (samples.txt)
//   metrics_to_json                 harness.cpp:154-175 (metrics.json, "rcs-metrics-v1")
// JSON is written the way nlohmann::json::dump(2) writes it (2-space indent,
// object keys in sorted order), by a small value type of our own.
// GCC 13 reports a spurious -Wmaybe-uninitialized inside std::variant<std::string, ...> copies
#pragma GCC diagnostic ignored "-Wmaybe-uninitialized"
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdio>
#include <functional>
#include <iterator>
#include <map>
#include <memory>
#include <sstream>
#include <variant>

#include "rcs_b200.hpp"

namespace rcs {
namespace {

// ---------------------------------------------------------------- JSON value
struct JVal;
using JArr = std::vector<JVal>;
using JObj = std::map<std::string, JVal>;
struct JVal {
    // null, bool, unsigned, signed, double, string, array, object
    std::variant<std::monostate, bool, std::uint64_t, std::int64_t, double, std::string, std::shared_ptr<JArr>,
                 std::shared_ptr<JObj>>
        v;
    JVal() = default;
    JVal(std::uint64_t x) : v(x) {}
    JVal(int x) : v(static_cast<std::int64_t>(x)) {}
    JVal(std::int64_t x) : v(x) {}
    JVal(double x) : v(x) {}
    JVal(const std::string& s) : v(s) {}
    JVal(const char* s) : v(std::string(s)) {}
    static JVal arr() {
        JVal j;
        j.v = std::make_shared<JArr>();
        return j;
    }
    static JVal obj() {
        JVal j;
        j.v = std::make_shared<JObj>();
        return j;
    }
    JArr& a() { return *std::get<std::shared_ptr<JArr>>(v); }
    const JArr& a() const { return *std::get<std::shared_ptr<JArr>>(v); }
    JObj& o() { return *std::get<std::shared_ptr<JObj>>(v); }
    const JObj& o() const { return *std::get<std::shared_ptr<JObj>>(v); }
    bool is_arr() const { return std::holds_alternative<std::shared_ptr<JArr>>(v); }
    bool is_obj() const { return std::holds_alternative<std::shared_ptr<JObj>>(v); }
    bool is_str() const { return std::holds_alternative<std::string>(v); }
    bool is_num() const {
        return std::holds_alternative<std::uint64_t>(v) || std::holds_alternative<std::int64_t>(v) ||
               std::holds_alternative<double>(v);
    }
    std::int64_t as_int() const {
        if (auto p = std::get_if<std::uint64_t>(&v)) return static_cast<std::int64_t>(*p);
        if (auto p = std::get_if<std::int64_t>(&v)) return *p;
        if (auto p = std::get_if<double>(&v)) return static_cast<std::int64_t>(*p);
        throw ConfigError("plan JSON: number expected");
    }
    const std::string& as_str() const {
        if (!is_str()) throw ConfigError("plan JSON: string expected");
        return std::get<std::string>(v);
    }
    JVal& operator[](const std::string& k) { return o()[k]; }
    const JVal& at(const std::string& k) const {
        auto it = o().find(k);
        if (it == o().end()) throw ConfigError("plan JSON: missing key \"" + k + "\"");
        return it->second;
    }
};

void dump_str(std::string& out, const std::string& s) {
    out += '"';
    for (unsigned char c : s) {
        switch (c) {
            case '"': out += "\\\""; break;
            case '\\': out += "\\\\"; break;
            case '\n': out += "\\n"; break;
            case '\t': out += "\\t"; break;
            case '\r': out += "\\r"; break;
            case '\b': out += "\\b"; break;
            case '\f': out += "\\f"; break;
            default:
                if (c < 0x20) {
                    char b[8];
                    std::snprintf(b, sizeof b, "\\u%04x", c);
                    out += b;
                } else {
                    out += static_cast<char>(c);
                }
        }
    }
    out += '"';
}

// nlohmann's double format: shortest round-trip digits ("%.17g" trimmed), ".0" for integral values
std::string dump_double(double x) {
    if (!std::isfinite(x)) return "null";
    char b[64];
    for (int prec = 1; prec <= 17; ++prec) {
        std::snprintf(b, sizeof b, "%.*g", prec, x);
        if (std::strtod(b, nullptr) == x) break;
    }
    std::string s = b;
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
    return s;
}

void dump(std::string& out, const JVal& j, int indent, int level) {
    const std::string pad(static_cast<std::size_t>(indent * (level + 1)), ' ');
    const std::string pad0(static_cast<std::size_t>(indent * level), ' ');
    if (std::holds_alternative<std::monostate>(j.v)) out += "null";
    else if (auto b = std::get_if<bool>(&j.v)) out += *b ? "true" : "false";
    else if (auto u = std::get_if<std::uint64_t>(&j.v)) out += std::to_string(*u);
    else if (auto i = std::get_if<std::int64_t>(&j.v)) out += std::to_string(*i);
    else if (auto d = std::get_if<double>(&j.v)) out += dump_double(*d);
    else if (j.is_str()) dump_str(out, j.as_str());
    else if (j.is_arr()) {
        const JArr& a = j.a();
        if (a.empty()) {
            out += "[]";
            return;
        }
        out += "[\n";
        for (std::size_t k = 0; k < a.size(); ++k) {
            out += pad;
            dump(out, a[k], indent, level + 1);
            out += k + 1 < a.size() ? ",\n" : "\n";
        }
        out += pad0 + "]";
    } else {
        const JObj& o = j.o();
        if (o.empty()) {
            out += "{}";
            return;
        }
        out += "{\n";
        std::size_t k = 0;
        for (const auto& [key, val] : o) {
            out += pad;
            dump_str(out, key);
            out += ": ";
            dump(out, val, indent, level + 1);
            out += ++k < o.size() ? ",\n" : "\n";
        }
        out += pad0 + "}";
    }
}

// minimal recursive-descent parser (objects, arrays, strings, numbers, literals)
struct Parser {
    const std::string& s;
    std::size_t i = 0;
    void ws() {
        while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
    }
    [[noreturn]] void fail(const char* what) {
        throw ConfigError(std::string("plan JSON: ") + what + " at offset " + std::to_string(i));
    }
    JVal value() {
        ws();
        if (i >= s.size()) fail("unexpected end");
        const char c = s[i];
        if (c == '{') {
            ++i;
            JVal j = JVal::obj();
            ws();
            if (i < s.size() && s[i] == '}') {
                ++i;
                return j;
            }
            for (;;) {
                ws();
                const std::string k = str();
                ws();
                if (i >= s.size() || s[i] != ':') fail("':' expected");
                ++i;
                j.o()[k] = value();
                ws();
                if (i < s.size() && s[i] == ',') {
                    ++i;
                    continue;
                }
                if (i < s.size() && s[i] == '}') {
                    ++i;
                    return j;
                }
                fail("',' or '}' expected");
            }
        }
        if (c == '[') {
            ++i;
            JVal j = JVal::arr();
            ws();
            if (i < s.size() && s[i] == ']') {
                ++i;
                return j;
            }
            for (;;) {
                j.a().push_back(value());
                ws();
                if (i < s.size() && s[i] == ',') {
                    ++i;
                    continue;
                }
                if (i < s.size() && s[i] == ']') {
                    ++i;
                    return j;
                }
                fail("',' or ']' expected");
            }
        }
        if (c == '"') return JVal(str());
        if (s.compare(i, 4, "null") == 0) {
            i += 4;
            return JVal();
        }
        if (s.compare(i, 4, "true") == 0) {
            i += 4;
            JVal j;
            j.v = true;
            return j;
        }
        if (s.compare(i, 5, "false") == 0) {
            i += 5;
            JVal j;
            j.v = false;
            return j;
        }
        const std::size_t b = i;
        while (i < s.size() && (std::isdigit(static_cast<unsigned char>(s[i])) || s[i] == '-' || s[i] == '+' ||
                                s[i] == '.' || s[i] == 'e' || s[i] == 'E'))
            ++i;
        if (b == i) fail("value expected");
        const std::string num = s.substr(b, i - b);
        if (num.find_first_of(".eE") != std::string::npos) return JVal(std::stod(num));
        if (num[0] == '-') return JVal(static_cast<std::int64_t>(std::stoll(num)));
        return JVal(static_cast<std::uint64_t>(std::stoull(num)));
    }
    std::string str() {
        if (i >= s.size() || s[i] != '"') fail("string expected");
        ++i;
        std::string out;
        while (i < s.size() && s[i] != '"') {
            char c = s[i++];
            if (c == '\\') {
                if (i >= s.size()) fail("bad escape");
                const char e = s[i++];
                switch (e) {
                    case 'n': c = '\n'; break;
                    case 't': c = '\t'; break;
                    case 'r': c = '\r'; break;
                    case 'b': c = '\b'; break;
                    case 'f': c = '\f'; break;
                    case 'u': c = static_cast<char>(std::stoi(s.substr(i, 4), nullptr, 16)); i += 4; break;
                    default: c = e;
                }
            }
            out += c;
        }
        if (i >= s.size()) fail("unterminated string");
        ++i;
        return out;
    }
};

JVal names_of(const TensorNetwork& net, const std::vector<Label>& labels) {
    JVal a = JVal::arr();
    for (Label l : labels) a.a().push_back(JVal(net.label_name(l)));
    return a;
}

}  // namespace

std::string plan_to_json(const ContractionPlan& plan, const TensorNetwork& network) {
    const int n_leaves = static_cast<int>(network.tensors.size());
    std::vector<JVal> rendered(n_leaves + plan.steps.size());
    for (int i = 0; i < n_leaves; ++i) rendered[i] = JVal(i);
    JVal order = JVal::arr();
    for (const PlanStep& s : plan.steps) {
        JVal pair = JVal::arr();
        pair.a().push_back(rendered.at(s.lhs));
        pair.a().push_back(rendered.at(s.rhs));
        rendered.at(s.result) = pair;
        order = pair;
    }
    JVal j = JVal::obj();
    j["order"] = order;
    j["sliced"] = names_of(network, plan.sliced);
    j["broken"] = names_of(network, plan.broken);
    JVal per = JVal::arr();
    for (const PlanStep& s : plan.steps) {
        JVal st = JVal::obj();
        JVal ops = JVal::arr();
        ops.a().push_back(JVal(s.lhs));
        ops.a().push_back(JVal(s.rhs));
        st["operands"] = ops;
        st["result_labels"] = names_of(network, s.result_labels);
        st["summed_indices"] = JVal(s.summed);
        st["flops"] = JVal(s.flops);
        st["result_bytes"] = JVal(s.result_bytes);
        per.a().push_back(st);
    }
    j["per_step"] = per;
    JVal tot = JVal::obj();
    tot["flops_per_slice"] = JVal(plan.flops_per_slice);
    tot["subtask_flops"] = JVal(plan.subtask_flops());
    tot["peak_bytes"] = JVal(plan.peak_bytes);
    tot["traffic_bytes_per_slice"] = JVal(plan.traffic_bytes_per_slice);
    tot["n_slices"] = JVal(plan.n_slices());
    tot["memory_budget_bytes"] = JVal(plan.memory_budget_bytes);
    j["totals"] = tot;
    std::string out;
    dump(out, j, 2, 0);
    return out;
}

ContractionPlan plan_from_json(const std::string& text, const TensorNetwork& network) {
    Parser ps{text};
    const JVal j = ps.value();
    if (!j.is_obj()) throw ConfigError("plan JSON: object expected");
    std::map<std::string, Label> by_name;
    for (std::size_t l = 0; l < network.label_names.size(); ++l) by_name[network.label_names[l]] = static_cast<Label>(l);
    auto labels_of = [&](const JVal& arr) {
        std::vector<Label> out;
        if (!arr.is_arr()) throw ConfigError("plan JSON: label list expected");
        for (const JVal& n : arr.a()) {
            auto it = by_name.find(n.as_str());
            if (it == by_name.end()) throw ConfigError("plan JSON: unknown label " + n.as_str());
            out.push_back(it->second);
        }
        return out;
    };
    ContractionPlan plan;
    plan.sliced = labels_of(j.at("sliced"));
    plan.broken = labels_of(j.at("broken"));
    for (Label l : network.output_labels)
        if (!network.is_open(l)) plan.fixed_outputs.push_back(l);
    if (j.o().count("totals") && j.at("totals").is_obj() && j.at("totals").o().count("memory_budget_bytes"))
        plan.memory_budget_bytes = static_cast<std::uint64_t>(j.at("totals").at("memory_budget_bytes").as_int());
    // label sets of the leaves with pinned (fixed output / broken / sliced) labels removed
    const int n_leaves = static_cast<int>(network.tensors.size());
    std::vector<char> removed(network.label_names.size(), 0);
    for (Label l : plan.fixed_outputs) removed[l] = 1;
    for (Label l : plan.broken) removed[l] = 1;
    for (Label l : plan.sliced) removed[l] = 1;
    std::vector<std::vector<Label>> sets;
    for (const Tensor& t : network.tensors) {
        std::vector<Label> v;
        for (Label l : t.labels)
            if (!removed[l]) v.push_back(l);
        std::sort(v.begin(), v.end());
        sets.push_back(std::move(v));
    }
    std::vector<char> used(n_leaves, 0);
    constexpr double kSat = 1.8446744073709552e19;
    auto sat = [&](double x) { return x >= kSat ? ~std::uint64_t{0} : static_cast<std::uint64_t>(x); };
    double live = 0, peak = 0, flops = 0, traffic = 0;
    std::vector<double> bytes;
    for (const auto& v : sets) {
        bytes.push_back(16.0 * std::ldexp(1.0, static_cast<int>(v.size())));
        live += bytes.back();
    }
    peak = live;
    // post-order over the nested pairs (left, right, node): the reference's step order
    std::function<int(const JVal&)> walk = [&](const JVal& node) -> int {
        if (node.is_num()) {
            const std::int64_t leaf = node.as_int();
            if (leaf < 0 || leaf >= n_leaves || used[leaf]) throw ConfigError("plan JSON: bad or repeated leaf");
            used[leaf] = 1;
            return static_cast<int>(leaf);
        }
        if (!node.is_arr() || node.a().size() != 2) throw ConfigError("plan JSON: order must nest pairs");
        const int a = walk(node.a()[0]);
        const int b = walk(node.a()[1]);
        std::vector<Label> res, shared;
        std::set_symmetric_difference(sets[a].begin(), sets[a].end(), sets[b].begin(), sets[b].end(),
                                      std::back_inserter(res));
        std::set_intersection(sets[a].begin(), sets[a].end(), sets[b].begin(), sets[b].end(),
                              std::back_inserter(shared));
        PlanStep st;
        st.lhs = a;
        st.rhs = b;
        st.result = n_leaves + static_cast<int>(plan.steps.size());
        st.result_labels = res;
        st.summed = shared.size();
        const double f = 8.0 * std::ldexp(1.0, static_cast<int>(res.size() + shared.size()));
        const double rb = 16.0 * std::ldexp(1.0, static_cast<int>(res.size()));
        st.flops = sat(f);
        st.result_bytes = sat(rb);
        const double io = bytes[a] + bytes[b] + rb;
        peak = std::max(peak, live + io);
        flops += f;
        traffic += io;
        live = std::max(0.0, live + rb - bytes[a] - bytes[b]);
        sets.push_back(std::move(res));
        bytes.push_back(rb);
        plan.steps.push_back(std::move(st));
        return plan.steps.back().result;
    };
    const JVal& order = j.at("order");
    if (!(order.is_arr() && order.a().empty())) walk(order);
    if (n_leaves > 1 && static_cast<int>(plan.steps.size()) != n_leaves - 1)
        throw ConfigError("plan JSON: order does not cover every leaf");
    // node ids: the writer's own ids when per_step carries them (the reference
    // numbers internal nodes by creation, not by step), else n_leaves + step
    if (j.o().count("per_step") && j.at("per_step").is_arr() && j.at("per_step").a().size() == plan.steps.size()) {
        const JArr& per = j.at("per_step").a();
        const int n_steps = static_cast<int>(plan.steps.size());
        std::vector<int> id(n_leaves + n_steps, -1);
        for (int i = 0; i < n_leaves; ++i) id[i] = i;
        for (int s = 0; s < n_steps; ++s) {
            const JVal& ops = per[s].at("operands");
            if (!ops.is_arr() || ops.a().size() != 2) throw ConfigError("plan JSON: operands must be pairs");
            const int kids[2] = {plan.steps[s].lhs, plan.steps[s].rhs};
            for (int side = 0; side < 2; ++side) {
                const std::int64_t want = ops.a()[side].as_int();
                if (kids[side] < n_leaves ? want != kids[side] : (id[kids[side]] = static_cast<int>(want), false))
                    throw ConfigError("plan JSON: per_step operands disagree with order");
            }
        }
        id[n_leaves + n_steps - 1] = n_leaves + n_steps - 1;  // the root: the last node created
        std::vector<char> seen(n_leaves + n_steps, 0);
        for (int v : id) {
            if (v < 0 || v >= n_leaves + n_steps || seen[v]) throw ConfigError("plan JSON: inconsistent node ids");
            seen[v] = 1;
        }
        for (PlanStep& st : plan.steps) {
            st.lhs = id[st.lhs];
            st.rhs = id[st.rhs];
            st.result = id[st.result];
        }
    }
    plan.flops_per_slice = sat(flops);
    plan.traffic_bytes_per_slice = sat(traffic);
    plan.peak_bytes = sat(peak);
    return plan;
}

std::string timings_to_csv(const std::vector<SubtaskTiming>& timings) {
    std::ostringstream out;
    out << "subtask_id,config_bits,wall_ms,flops\n";
    for (const SubtaskTiming& t : timings)
        out << t.subtask_id << ',' << t.config_bits << ',' << t.wall_ms << ',' << t.flops << '\n';
    return out.str();
}

std::string samples_to_text(const SampleSet& samples) {
    std::ostringstream out;
    out << "# provenance=" << (samples.provenance == Provenance::TopK ? "top_k" : "direct") << "\n";
    if (samples.provenance == Provenance::TopK) out << "# k=" << samples.k << "\n";
    out << "# n_qubits=" << samples.n_qubits << "\n";
    for (std::uint64_t s : samples.bitstrings) {
        std::string line(static_cast<std::size_t>(samples.n_qubits), '0');
        for (int q = 0; q < samples.n_qubits; ++q)
            if ((s >> q) & 1) line[static_cast<std::size_t>(q)] = '1';
        out << line << '\n';
    }
    return out.str();
}

SampleSet samples_from_text(const std::string& text) {
    SampleSet samples;
    std::istringstream in(text);
    std::string line;
    while (std::getline(in, line)) {
        if (line.empty()) continue;
        if (line[0] == '#') {
            if (line.rfind("# provenance=top_k", 0) == 0) samples.provenance = Provenance::TopK;
            else if (line.rfind("# k=", 0) == 0) samples.k = std::stoull(line.substr(4));
            else if (line.rfind("# n_qubits=", 0) == 0) samples.n_qubits = std::stoi(line.substr(11));
            continue;
        }
        std::uint64_t index = 0;
        for (std::size_t q = 0; q < line.size(); ++q)
            if (line[q] == '1') index |= std::uint64_t{1} << q;
        if (samples.n_qubits == 0) samples.n_qubits = static_cast<int>(line.size());
        samples.bitstrings.push_back(index);
    }
    return samples;
}

std::string metrics_to_json(const MetricsReport& m, const MetricsInputs& c) {
    JVal j = JVal::obj();
    j["schema"] = JVal("rcs-metrics-v1");
    j["xeb"] = JVal(m.xeb);
    j["fidelity"] = JVal(m.fidelity);
    j["predicted_xeb"] = JVal(m.predicted_xeb);
    j["pearson_r"] = JVal(m.pearson_r);
    j["pt_ks_statistic"] = JVal(m.pt_ks_statistic);
    j["pt_p_value"] = JVal(m.pt_p_value);
    j["xeb_over_fidelity"] = JVal(m.xeb_over_fidelity);
    JVal in = JVal::obj();
    in["n_qubits"] = JVal(c.n_qubits);
    in["n_cycles"] = JVal(c.n_cycles);
    in["topology"] = JVal(c.topology);
    in["seed"] = JVal(c.seed);
    in["l"] = JVal(static_cast<std::uint64_t>(c.l));
    in["M"] = JVal(c.n_groups);
    in["K"] = JVal(c.broken_edges);
    in["m"] = JVal(c.m_configs);
    in["k"] = JVal(c.k);
    in["sample_mode"] = JVal(c.sample_mode);
    j["inputs"] = in;
    std::string out;
    dump(out, j, 2, 0);
    return out;
}

}  // namespace rcs
