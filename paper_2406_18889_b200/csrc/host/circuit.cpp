// Circuit model and network builder (host side, input to the hot path).
//
// Semantics follow the reference exactly so that the same (n, cycles,
// topology, seed) yields the same gates, labels and leaf data:
//   gate unitaries           circuit.cpp:33-61
//   line/ring/grid patterns  circuit.cpp:65-110   (+ "sycamore53", new)
//   random circuit           circuit.cpp:112-161 (one RNG draw per 1q slot)
//   circuit_to_network      tensor_network.cpp:20-92
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <set>

#include "rcs_b200.hpp"

namespace rcs {

// ---------------------------------------------------------------- RNG
std::uint64_t Rng::next_u64() {
    s_ += 0x9e3779b97f4a7c15ull;
    std::uint64_t z = s_;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
double Rng::next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
std::uint64_t Rng::next_below(std::uint64_t bound) {
    const std::uint64_t reject_below = (0 - bound) % bound;
    std::uint64_t r = next_u64();
    while (r < reject_below) r = next_u64();
    return r % bound;
}
Rng Rng::split(std::uint64_t tag) const {
    std::uint64_t z = s_ ^ (tag * 0xd6e8feb86659fd93ull + 0xa3c59ac2f0ull);
    z = (z ^ (z >> 32)) * 0xd6e8feb86659fd93ull;
    return Rng(z ^ (z >> 32));
}

// ---------------------------------------------------------------- gates
const char* gate_kind_name(GateKind kind) {
    static const char* names[] = {"sqrt_x", "sqrt_y", "sqrt_w", "fsim"};
    return names[static_cast<int>(kind)];
}

GateKind gate_kind_from_name(const std::string& name) {
    for (int k = 0; k < 4; ++k)
        if (name == gate_kind_name(static_cast<GateKind>(k))) return static_cast<GateKind>(k);
    throw ConfigError("unknown gate kind: " + name);
}

std::vector<cplx> gate_unitary(GateKind kind) {
    const cplx I(0.0, 1.0);
    const cplx p = 0.5 * (1.0 + I), m = 0.5 * (1.0 - I);
    if (kind == GateKind::SqrtX) return {p, m, m, p};
    if (kind == GateKind::SqrtY) return {p, 0.5 * (-1.0 - I), p, p};
    if (kind == GateKind::SqrtW) {
        const double r = std::sqrt(2.0);
        return {p, -I / r, 1.0 / r, p};
    }
    // fSim(theta = pi/2, phi = pi/6): |01>,|10> swap with -i sin(theta), |11> phase
    const double theta = M_PI / 2.0, phi = M_PI / 6.0;
    const cplx c = std::cos(theta);
    const cplx s = -I * std::sin(theta);
    const cplx e = std::exp(-I * phi);
    std::vector<cplx> u(16, cplx(0.0, 0.0));
    u[0] = 1.0;
    u[5] = c;
    u[6] = s;
    u[9] = s;
    u[10] = c;
    u[15] = e;
    return u;
}

// ---------------------------------------------------------------- topologies
namespace {

void add_chain(std::vector<std::pair<int, int>>& out, int n, int first) {
    for (int q = first; q + 1 < n; q += 2) out.emplace_back(q, q + 1);
}

// Diagonal ("rotated square") lattice of rows x cols sites, as on Google's
// Sycamore and USTC's Zuchongzhi chips.  Site (r, c) couples to (r+1, c) and
// (r+1, c -/+ 1) depending on row parity; the four coupler classes A,B,C,D follow
// the row parity and the direction; the cycle order is the supremacy sequence
// ABCDCDAB.  Sites in `missing` do not exist; qubits are numbered row-major over
// the remaining sites.
Topology diagonal_lattice(int rows, int cols, const std::vector<int>& missing, int n_qubits,
                          const char* name) {
    std::vector<int> id(rows * cols, -1);
    int next = 0;
    for (int s = 0; s < rows * cols; ++s)
        if (std::find(missing.begin(), missing.end(), s) == missing.end()) id[s] = next++;
    if (n_qubits != next) throw ConfigError(std::string(name) + " needs n_qubits=" + std::to_string(next));
    Topology t;
    t.patterns.assign(4, {});
    for (int r = 0; r + 1 < rows; ++r)
        for (int c = 0; c < cols; ++c) {
            const int a = id[r * cols + c];
            if (a < 0) continue;
            const int cl = (r % 2 == 0) ? c : c - 1;
            const int cr = (r % 2 == 0) ? c + 1 : c;
            if (cl >= 0 && cl < cols) {
                const int b = id[(r + 1) * cols + cl];
                if (b >= 0) t.patterns[(r % 2 == 0) ? 0 : 1].emplace_back(a, b);
            }
            if (cr >= 0 && cr < cols) {
                const int b = id[(r + 1) * cols + cr];
                if (b >= 0) t.patterns[(r % 2 == 0) ? 2 : 3].emplace_back(a, b);
            }
        }
    t.sequence = {0, 1, 2, 3, 2, 3, 0, 1};
    return t;
}

// Google Sycamore-53: 9 x 6 sites with the one broken site (0, 3) removed.
Topology sycamore(int n_qubits) { return diagonal_lattice(9, 6, {3}, n_qubits, "sycamore53"); }

// Zuchongzhi-style 60 qubits (BASELINE cfg5): the 66-site 11 x 6 lattice of
// Zuchongzhi 2.x, with the 60 qubits of its first 10 rows in use.
Topology zuchongzhi60(int n_qubits) { return diagonal_lattice(10, 6, {}, n_qubits, "zuchongzhi60"); }

}  // namespace

Topology make_topology(const std::string& name, int n_qubits) {
    Topology t;
    if (name == "line" || name == "ring") {
        t.patterns.resize(2);
        add_chain(t.patterns[0], n_qubits, 0);
        add_chain(t.patterns[1], n_qubits, 1);
        if (name == "ring" && n_qubits >= 3 && n_qubits % 2 == 0)
            t.patterns[1].emplace_back(n_qubits - 1, 0);
        t.sequence = {0, 1};
    } else if (name.rfind("grid(", 0) == 0) {
        int R = 0, Cc = 0;
        if (std::sscanf(name.c_str(), "grid(%d,%d)", &R, &Cc) != 2 || R < 1 || Cc < 1)
            throw ConfigError("bad grid topology spec: " + name);
        if (R * Cc != n_qubits) throw ConfigError("grid dimensions do not match qubit count");
        t.patterns.resize(4);
        for (int r = 0; r + 1 < R; ++r)
            for (int c = 0; c < Cc; ++c) t.patterns[r % 2].emplace_back(r * Cc + c, (r + 1) * Cc + c);
        for (int r = 0; r < R; ++r)
            for (int c = 0; c + 1 < Cc; ++c)
                t.patterns[2 + c % 2].emplace_back(r * Cc + c, r * Cc + c + 1);
        t.sequence = {0, 1, 2, 3, 2, 3, 0, 1};
    } else if (name == "sycamore53") {
        t = sycamore(n_qubits);
    } else if (name == "zuchongzhi60") {
        t = zuchongzhi60(n_qubits);
    } else {
        throw ConfigError("unknown topology: " + name);
    }
    t.name = name;
    t.n_qubits = n_qubits;
    bool any = false;
    for (const auto& p : t.patterns) any = any || !p.empty();
    if (!any)
        throw ConfigError("topology has no couplers for n_qubits=" + std::to_string(n_qubits));
    return t;
}

Circuit gen_random_circuit(int n_qubits, int n_cycles, const std::string& topology,
                           std::uint64_t seed) {
    if (n_qubits < 2) throw ConfigError("n_qubits must be >= 2");
    if (n_cycles < 1) throw ConfigError("n_cycles must be >= 1");
    const Topology topo = make_topology(topology, n_qubits);
    Circuit circ;
    circ.n_qubits = n_qubits;
    circ.seed = seed;
    circ.topology = topology;
    circ.exceeds_exact_cap = n_qubits > 24;
    Rng rng(seed);
    std::vector<int> last(n_qubits, -1);  // previous single-qubit kind per qubit
    const std::vector<cplx> fsim = gate_unitary(GateKind::TwoQubit);
    for (int cyc = 0; cyc < n_cycles; ++cyc) {
        Layer ones;
        ones.gates.reserve(n_qubits);
        for (int q = 0; q < n_qubits; ++q) {
            // one draw per slot over the kinds that differ from the previous one
            const int choices = last[q] < 0 ? 3 : 2;
            int pick = static_cast<int>(rng.next_below(choices));
            int kind = 0;
            for (; kind < 3; ++kind) {
                if (kind == last[q]) continue;
                if (pick-- == 0) break;
            }
            last[q] = kind;
            const GateKind gk = static_cast<GateKind>(kind);
            ones.gates.push_back(Gate{gk, {q}, gate_unitary(gk)});
        }
        circ.layers.push_back(std::move(ones));
        Layer twos;
        for (const auto& [a, b] : topo.patterns[topo.sequence[cyc % topo.sequence.size()]])
            twos.gates.push_back(Gate{GateKind::TwoQubit, {a, b}, fsim});
        circ.layers.push_back(std::move(twos));
    }
    return circ;
}

// ---------------------------------------------------------------- network
Label TensorNetwork::label_by_name(const std::string& name) const {
    for (std::size_t i = 0; i < label_names.size(); ++i)
        if (label_names[i] == name) return static_cast<Label>(i);
    throw ConfigError("unknown index label: " + name);
}

bool TensorNetwork::is_open(Label l) const {
    for (Label o : open_labels)
        if (o == l) return true;
    return false;
}

TensorNetwork circuit_to_network(const Circuit& circuit, const std::vector<int>& open_qubits) {
    const std::set<int> open(open_qubits.begin(), open_qubits.end());
    if (open.size() != open_qubits.size()) throw ConfigError("duplicate open qubits");
    for (int q : open_qubits)
        if (q < 0 || q >= circuit.n_qubits)
            throw ConfigError("open qubit out of range: " + std::to_string(q));
    TensorNetwork net;
    net.n_qubits = circuit.n_qubits;
    net.n_layers = static_cast<int>(circuit.layers.size());
    auto fresh = [&net](int q, const std::string& suffix) {
        net.label_names.push_back("q" + std::to_string(q) + "." + suffix);
        return static_cast<Label>(net.label_names.size() - 1);
    };
    std::vector<Label> wire(circuit.n_qubits);
    std::vector<int> born(circuit.n_qubits, -1);  // layer that produced the current wire
    for (int q = 0; q < circuit.n_qubits; ++q) {  // |0> cap on every input leg
        wire[q] = fresh(q, "in");
        net.tensors.push_back(Tensor{{wire[q]}, {cplx(1.0, 0.0), cplx(0.0, 0.0)}});
    }
    for (int t = 0; t < net.n_layers; ++t) {
        for (const Gate& g : circuit.layers[t].gates) {
            Tensor tensor;
            tensor.data = g.unitary;
            std::vector<Label> outs;
            for (int q : g.targets) {
                if (born[q] >= 0) net.wire_edges.push_back({wire[q], q, born[q]});
                outs.push_back(fresh(q, "t" + std::to_string(t)));
            }
            // labels = outputs then inputs, so index = U[out][in] row-major
            tensor.labels = outs;
            for (int q : g.targets) tensor.labels.push_back(wire[q]);
            for (std::size_t j = 0; j < g.targets.size(); ++j) {
                wire[g.targets[j]] = outs[j];
                born[g.targets[j]] = t;
            }
            net.tensors.push_back(std::move(tensor));
        }
    }
    net.output_labels = wire;
    for (int q = 0; q < circuit.n_qubits; ++q)
        if (open.count(q)) {
            net.open_qubits.push_back(q);
            net.open_labels.push_back(wire[q]);
        }
    return net;
}

}  // namespace rcs
