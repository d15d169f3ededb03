// Contraction-path planner at scale, new work.
//
// The reference planner (contraction_plan.cpp:85-377, restated bit for bit in
// planner.cpp) keeps uint64 costs that wrap at rank >= 60, grows one greedy tree,
// and slices by peak memory until it stalls; on Sycamore-scale circuits it
// cannot produce a plan.  This planner keeps the reference's output
// format (ContractionPlan: post-order PlanSteps over the original leaves, sliced
// labels, per-slice totals) and replaces the search:
//
//   * costs in the log2 domain (double), so nothing overflows;
//   * batch-aware cost model: a node that holds the projections of b fixed
//     output qubits exists in min(M, 2^b) group variants (the executor's
//     sparse-state batching), so its size and step cost carry that factor;
//   * simplification: tensors of rank <= 2 (single-qubit gates, |0> caps,
//     projected outputs) are folded into a neighbour first;
//   * hyper-optimised trials on all host threads: recursive multilevel
//     Fiduccia-Mattheyses bisection of the tensor graph (imbalance and cutoff
//     drawn per trial; each part's tensor rank is its cut), finished below the
//     cutoff - and in a quarter of the trials for the whole network - by a
//     randomized greedy (cost = size(ab) - alpha (size(a) + size(b)) with
//     Gumbel noise at temperature T, alpha and T drawn per trial);
//   * stem-aware slicing: while the widest tensor exceeds the budget, slice the
//     label of the widest tensor that minimises the total cost, where steps
//     whose subtree holds no sliced label run once (the executor caches them)
//     and the others run once per slice;
//   * subtree reconfiguration: every subtree cut at up to 8 inputs is
//     re-contracted optimally by dynamic programming over input subsets, under
//     the same sliced cost and width limit, repeated until nothing improves.
//
// Budget semantics: the widest tensor (including group variants) at 16 B per
// amplitude must fit in memory_budget_bytes / 4 (operands + result + slack).
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <bit>
#include <array>
#include <chrono>
#include <functional>
#include <cmath>
#include <limits>
#include <mutex>
#include <numeric>
#include <queue>
#include <random>
#include <thread>

#include "rcs_b200.hpp"

namespace rcs {
namespace {

// ---------------------------------------------------------------- label sets
struct LSet {
    std::vector<std::uint64_t> w;
    LSet() = default;
    explicit LSet(int n) : w((n + 63) / 64, 0) {}
    void set(int i) { w[i >> 6] |= std::uint64_t{1} << (i & 63); }
    void reset(int i) { w[i >> 6] &= ~(std::uint64_t{1} << (i & 63)); }
    bool has(int i) const { return (w[i >> 6] >> (i & 63)) & 1; }
    int count() const {
        int c = 0;
        for (auto x : w) c += std::popcount(x);
        return c;
    }
    void xor_in(const LSet& o) {
        for (std::size_t i = 0; i < w.size(); ++i) w[i] ^= o.w[i];
    }
    int union_count(const LSet& o) const {
        int c = 0;
        for (std::size_t i = 0; i < w.size(); ++i) c += std::popcount(w[i] | o.w[i]);
        return c;
    }
    int and_count(const LSet& o) const {
        int c = 0;
        for (std::size_t i = 0; i < w.size(); ++i) c += std::popcount(w[i] & o.w[i]);
        return c;
    }
    bool intersects(const LSet& o) const {
        for (std::size_t i = 0; i < w.size(); ++i)
            if (w[i] & o.w[i]) return true;
        return false;
    }
    template <class F>
    void each(F&& f) const {
        for (std::size_t i = 0; i < w.size(); ++i)
            for (std::uint64_t x = w[i]; x; x &= x - 1) f(static_cast<int>(i * 64 + std::countr_zero(x)));
    }
};

// ---------------------------------------------------------------- the problem
struct Problem {
    int n_labels = 0;
    int n_leaves = 0;
    std::vector<LSet> leaf;      // leaf label sets (fixed outputs and broken labels removed)
    std::vector<int> leaf_out;   // projected (fixed) output legs per leaf: group-variant bits
    LSet open;                   // open output labels: never sliced
    double log_m = 0;            // log2 of the group batch the plan is costed for
    double width = 0;            // max log2 size (rank + variant bits) per tensor
};

// A binary tree over the leaves: nodes [0, n_leaves) are leaves, the rest are
// internal with children (l, r); root = last node.
struct Tree {
    std::vector<int> l, r;  // -1 for leaves
    int root = -1;
};

// Per-node quantities of a tree under a sliced set.
struct Eval {
    std::vector<LSet> labels;   // output labels (sliced removed)
    std::vector<LSet> sub;      // all labels met in the subtree's leaves
    std::vector<int> var;       // variant bits
    std::vector<double> cost;   // log2 of the step's FLOPs (8 per complex MAC); leaves: -inf
    std::vector<char> dep;      // subtree holds a sliced label (runs once per slice)
    double total = 0;           // total cost of all slices (FLOP-equivalents of step_cost, linear)
    double flops = 0;           // total FLOPs of all slices
    double max_size = 0;        // max log2 size over nodes
};

double vbits(const Problem& pb, int outs) { return std::min<double>(pb.log_m, outs); }

// Step cost in FLOP-equivalents, the executor's time model: max(FLOPs, ridge x
// bytes), with the operands and the result read / written once at 8 B per
// complex element (tf32 storage) - the tcgen05 GEMMs are tensor-bound above the
// ridge and HBM-bound below it.  Off by default (FLOPs only): with every operand
// charged at HBM rates (ridge 128, RCSG_PLAN_RIDGE=128) the search on Sycamore-53
// m = 20 traded 3x more FLOPs for fewer narrow steps, more than the measured
// efficiency gap can repay - most small intermediates stay in the 126 MB L2.
double plan_ridge() {
    static const double r = getenv("RCSG_PLAN_RIDGE") ? atof(getenv("RCSG_PLAN_RIDGE")) : 0.0;
    return r;
}
double step_cost(double flops_log2, double sa, double sb, double sc, double r = plan_ridge()) {
    const double f = std::exp2(flops_log2);
    if (r <= 0) return f;
    return std::max(f, r * 8.0 * (std::exp2(sa) + std::exp2(sb) + std::exp2(sc)));
}

// post-order of internal nodes (children before parents)
std::vector<int> post_order(const Tree& t) {
    std::vector<int> out;
    std::vector<std::pair<int, int>> st{{t.root, 0}};
    while (!st.empty()) {
        auto& [v, s] = st.back();
        if (t.l[v] < 0) {
            st.pop_back();
            continue;
        }
        if (s == 0) {
            s = 1;
            st.push_back({t.l[v], 0});
        } else if (s == 1) {
            s = 2;
            st.push_back({t.r[v], 0});
        } else {
            out.push_back(v);
            st.pop_back();
        }
    }
    return out;
}

Eval evaluate(const Problem& pb, const Tree& t, const LSet& sliced, int n_sliced) {
    const int n = static_cast<int>(t.l.size());
    Eval e;
    e.labels.assign(n, LSet(pb.n_labels));
    e.sub.assign(n, LSet(pb.n_labels));
    e.var.assign(n, 0);
    e.cost.assign(n, -std::numeric_limits<double>::infinity());
    e.dep.assign(n, 0);
    std::vector<int> outs(n, 0);
    for (int i = 0; i < pb.n_leaves; ++i) {
        e.labels[i] = pb.leaf[i];
        e.sub[i] = pb.leaf[i];
        for (std::size_t k = 0; k < sliced.w.size(); ++k) e.labels[i].w[k] &= ~sliced.w[k];
        outs[i] = pb.leaf_out[i];
        e.var[i] = static_cast<int>(vbits(pb, outs[i]));
        e.dep[i] = pb.leaf[i].intersects(sliced);
        e.max_size = std::max(e.max_size, e.labels[i].count() + static_cast<double>(e.var[i]));
    }
    const double mult = std::ldexp(1.0, n_sliced);
    for (int v : post_order(t)) {
        const int a = t.l[v], b = t.r[v];
        const int uni = e.labels[a].union_count(e.labels[b]);
        e.labels[v] = e.labels[a];
        e.labels[v].xor_in(e.labels[b]);
        e.sub[v] = e.sub[a];
        for (std::size_t k = 0; k < e.sub[v].w.size(); ++k) e.sub[v].w[k] |= e.sub[b].w[k];
        outs[v] = outs[a] + outs[b];
        e.var[v] = static_cast<int>(vbits(pb, outs[v]));
        e.dep[v] = e.dep[a] || e.dep[b];
        const double fl = uni + e.var[v] + 3.0;
        e.cost[v] = std::log2(step_cost(fl, e.labels[a].count() + e.var[a], e.labels[b].count() + e.var[b],
                                        e.labels[v].count() + e.var[v]));
        e.total += std::exp2(e.cost[v]) * (e.dep[v] ? mult : 1.0);
        e.flops += std::exp2(fl) * (e.dep[v] ? mult : 1.0);
        e.max_size = std::max(e.max_size, e.labels[v].count() + static_cast<double>(e.var[v]));
    }
    return e;
}

// ---------------------------------------------------------------- simplification
// Folds every tensor of rank <= 2 into the neighbour that gives the smallest
// result; returns the reduced nodes as subtrees over the leaves.
struct Reduced {
    std::vector<int> node;    // tree node id of each reduced tensor
    std::vector<LSet> labels;
    std::vector<int> outs;
};

Reduced simplify(const Problem& pb, Tree& t) {
    Reduced rd;
    std::vector<char> live(pb.n_leaves, 1);
    std::vector<int> node(pb.n_leaves);
    std::iota(node.begin(), node.end(), 0);
    std::vector<LSet> lab = pb.leaf;
    std::vector<int> outs = pb.leaf_out;
    std::vector<std::vector<int>> holders(pb.n_labels);
    for (int i = 0; i < pb.n_leaves; ++i) lab[i].each([&](int l) { holders[l].push_back(i); });
    auto neighbours = [&](int x) {
        std::vector<int> nb;
        lab[x].each([&](int l) {
            for (int h : holders[l])
                if (h != x && live[h] && std::find(nb.begin(), nb.end(), h) == nb.end()) nb.push_back(h);
        });
        return nb;
    };
    bool changed = true;
    while (changed) {
        changed = false;
        for (int x = 0; x < pb.n_leaves; ++x) {
            if (!live[x] || lab[x].count() > 2) continue;
            const auto nb = neighbours(x);
            if (nb.empty()) continue;
            int best = -1, best_rank = 1 << 30;
            for (int y : nb) {
                LSet u = lab[y];
                u.xor_in(lab[x]);
                const int rk = u.count();
                if (rk < best_rank || (rk == best_rank && y < best)) {
                    best_rank = rk;
                    best = y;
                }
            }
            // merge x into best: new tree node (best, x)
            t.l.push_back(node[best]);
            t.r.push_back(node[x]);
            node[best] = static_cast<int>(t.l.size()) - 1;
            lab[x].each([&](int l) {
                auto& h = holders[l];
                h.erase(std::remove(h.begin(), h.end(), x), h.end());
                if (lab[best].has(l)) h.erase(std::remove(h.begin(), h.end(), best), h.end());  // contracted
                else h.push_back(best);
            });
            lab[best].xor_in(lab[x]);
            outs[best] += outs[x];
            live[x] = 0;
            changed = true;
        }
    }
    for (int x = 0; x < pb.n_leaves; ++x)
        if (live[x]) {
            rd.node.push_back(node[x]);
            rd.labels.push_back(lab[x]);
            rd.outs.push_back(outs[x]);
        }
    return rd;
}

// ---------------------------------------------------------------- greedy trials
struct GreedyParams {
    double alpha = 1.0;
    double temp = 0.0;
    std::uint64_t seed = 0;
};

// Randomized greedy over a subset of the reduced tensors (labels shared with
// tensors outside the subset stay open); appends internal nodes to `t` and
// returns the subtree's root node id.
int greedy_subset(const Problem& pb, const Reduced& rd, const std::vector<int>& members, Tree& t,
                  const GreedyParams& gp) {
    const int n0 = static_cast<int>(members.size());
    std::vector<LSet> lab(n0);
    std::vector<int> outs(n0), node(n0);
    for (int i = 0; i < n0; ++i) {
        lab[i] = rd.labels[members[i]];
        outs[i] = rd.outs[members[i]];
        node[i] = rd.node[members[i]];
    }
    std::vector<char> live(n0, 1);
    std::vector<int> version(n0, 0);
    std::vector<std::vector<int>> holders(pb.n_labels);
    for (int i = 0; i < n0; ++i) lab[i].each([&](int l) { holders[l].push_back(i); });
    std::mt19937_64 rng(gp.seed);
    std::uniform_real_distribution<double> U(1e-12, 1.0);
    auto lsize = [&](int rank, int o) { return rank + vbits(pb, o); };
    struct Cand {
        double key;
        int a, b, va, vb;
        bool operator>(const Cand& o) const { return key > o.key || (key == o.key && (a > o.a || (a == o.a && b > o.b))); }
    };
    std::priority_queue<Cand, std::vector<Cand>, std::greater<Cand>> pq;
    auto offer = [&](int a, int b) {
        if (a > b) std::swap(a, b);
        LSet u = lab[a];
        u.xor_in(lab[b]);
        const double sab = std::exp2(lsize(u.count(), outs[a] + outs[b]));
        const double sa = std::exp2(lsize(lab[a].count(), outs[a])), sb = std::exp2(lsize(lab[b].count(), outs[b]));
        const double c = sab - gp.alpha * (sa + sb);
        double key = (c >= 0 ? 1.0 : -1.0) * std::log2(1.0 + std::fabs(c));
        if (gp.temp > 0) key -= gp.temp * -std::log(-std::log(U(rng)));
        pq.push({key, a, b, version[a], version[b]});
    };
    for (int i = 0; i < n0; ++i)
        lab[i].each([&](int l) {
            if (holders[l].size() == 2 && holders[l][0] == i) offer(holders[l][0], holders[l][1]);
        });
    int n_live = n0;
    auto merge = [&](int a, int b) {
        // result stored in slot a
        t.l.push_back(node[a]);
        t.r.push_back(node[b]);
        node[a] = static_cast<int>(t.l.size()) - 1;
        lab[b].each([&](int l) {
            auto& h = holders[l];
            h.erase(std::remove(h.begin(), h.end(), b), h.end());
            if (lab[a].has(l)) h.erase(std::remove(h.begin(), h.end(), a), h.end());
            else h.push_back(a);
        });
        lab[a].xor_in(lab[b]);
        outs[a] += outs[b];
        live[b] = 0;
        ++version[a];
        ++version[b];
        --n_live;
        std::vector<int> nb;
        lab[a].each([&](int l) {
            for (int h : holders[l])
                if (h != a && std::find(nb.begin(), nb.end(), h) == nb.end()) nb.push_back(h);
        });
        for (int h : nb) offer(a, h);
    };
    while (!pq.empty()) {
        const Cand c = pq.top();
        pq.pop();
        if (!live[c.a] || !live[c.b] || version[c.a] != c.va || version[c.b] != c.vb) continue;
        merge(c.a, c.b);
    }
    // disconnected remainders: outer products, smallest first
    while (n_live > 1) {
        int a = -1, b = -1;
        double sa = 1e300, sb = 1e300;
        for (int i = 0; i < n0; ++i) {
            if (!live[i]) continue;
            const double sz = lsize(lab[i].count(), outs[i]);
            if (sz < sa) {
                b = a;
                sb = sa;
                a = i;
                sa = sz;
            } else if (sz < sb) {
                b = i;
                sb = sz;
            }
        }
        merge(std::min(a, b), std::max(a, b));
    }
    for (int i = 0; i < n0; ++i)
        if (live[i]) return node[i];
    return -1;
}

void greedy(const Problem& pb, const Reduced& rd, Tree& t, const GreedyParams& gp) {
    std::vector<int> all(rd.node.size());
    std::iota(all.begin(), all.end(), 0);
    t.root = greedy_subset(pb, rd, all, t, gp);
}

// ---------------------------------------------------------------- partitioning
// Multilevel Fiduccia-Mattheyses bisection of the tensor graph (edge weight =
// labels shared), recursive: each part's tensor has rank = its cut, so small
// balanced cuts make narrow trees (the hypergraph-partitioning route to good
// contraction trees for circuits).
struct Graph {
    std::vector<int> vw;                                  // node weights
    std::vector<std::vector<std::pair<int, int>>> adj;    // (neighbour, weight)
    int n() const { return static_cast<int>(vw.size()); }
};

long cut_of(const Graph& g, const std::vector<char>& side) {
    long c = 0;
    for (int v = 0; v < g.n(); ++v)
        for (auto [u, w] : g.adj[v])
            if (u > v && side[u] != side[v]) c += w;
    return c;
}

void fm_refine(const Graph& g, std::vector<char>& side, double eps, int max_passes = 8) {
    const int n = g.n();
    long W = 0;
    for (int w : g.vw) W += w;
    int max_vw = 1;
    for (int w : g.vw) max_vw = std::max(max_vw, w);
    const double cap = std::max((1.0 + eps) * W / 2.0, W / 2.0 + max_vw);  // at least one node of slack
    std::vector<long> gain(n);
    for (int pass = 0; pass < max_passes; ++pass) {
        long ws[2] = {0, 0};
        for (int v = 0; v < n; ++v) ws[static_cast<int>(side[v])] += g.vw[v];
        for (int v = 0; v < n; ++v) {
            long gv = 0;
            for (auto [u, w] : g.adj[v]) gv += side[u] != side[v] ? w : -w;
            gain[v] = gv;
        }
        std::vector<char> locked(n, 0);
        std::vector<int> moves;
        long cum = 0, best = 0;
        int best_len = 0;
        for (int step = 0; step < n; ++step) {
            int pick = -1;
            for (int v = 0; v < n; ++v) {
                if (locked[v]) continue;
                const int to = 1 - side[v];
                if (ws[to] + g.vw[v] > cap) continue;
                if (pick < 0 || gain[v] > gain[pick]) pick = v;
            }
            if (pick < 0) break;
            const int from = side[pick], to = 1 - from;
            side[pick] = static_cast<char>(to);
            ws[from] -= g.vw[pick];
            ws[to] += g.vw[pick];
            locked[pick] = 1;
            cum += gain[pick];
            for (auto [u, w] : g.adj[pick]) gain[u] += side[u] == to ? -2 * w : 2 * w;
            gain[pick] = -gain[pick];
            moves.push_back(pick);
            if (cum > best) {
                best = cum;
                best_len = static_cast<int>(moves.size());
            }
        }
        for (int i = static_cast<int>(moves.size()) - 1; i >= best_len; --i) side[moves[i]] ^= 1;
        if (best <= 0) break;
    }
}

// heavy-edge matching: coarse graph + fine -> coarse map
Graph coarsen(const Graph& g, std::vector<int>& map, std::mt19937_64& rng) {
    const int n = g.n();
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::shuffle(order.begin(), order.end(), rng);
    map.assign(n, -1);
    int nc = 0;
    for (int v : order) {
        if (map[v] >= 0) continue;
        int best = -1, bw = 0;
        for (auto [u, w] : g.adj[v])
            if (map[u] < 0 && u != v && w > bw) {
                bw = w;
                best = u;
            }
        map[v] = nc;
        if (best >= 0) map[best] = nc;
        ++nc;
    }
    Graph c;
    c.vw.assign(nc, 0);
    c.adj.assign(nc, {});
    for (int v = 0; v < n; ++v) c.vw[map[v]] += g.vw[v];
    std::vector<int> slot(nc, -1);
    for (int cv = 0; cv < nc; ++cv) (void)cv;
    std::vector<std::vector<int>> members(nc);
    for (int v = 0; v < n; ++v) members[map[v]].push_back(v);
    for (int cv = 0; cv < nc; ++cv) {
        auto& out = c.adj[cv];
        for (int v : members[cv])
            for (auto [u, w] : g.adj[v]) {
                const int cu = map[u];
                if (cu == cv) continue;
                if (slot[cu] < 0) {
                    slot[cu] = static_cast<int>(out.size());
                    out.push_back({cu, 0});
                }
                out[slot[cu]].second += w;
            }
        for (auto& [cu, w] : out) slot[cu] = -1;
    }
    return c;
}

std::vector<char> bisect_graph(const Graph& g, double eps, std::mt19937_64& rng) {
    const int n = g.n();
    if (n <= 48) {
        std::vector<char> best_side;
        long best_cut = -1;
        for (int rep = 0; rep < 6; ++rep) {
            std::vector<int> order(n);
            std::iota(order.begin(), order.end(), 0);
            std::shuffle(order.begin(), order.end(), rng);
            std::vector<char> side(n, 0);
            long ws[2] = {0, 0};
            for (int v : order) {
                const int s2 = ws[0] <= ws[1] ? 0 : 1;
                side[v] = static_cast<char>(s2);
                ws[s2] += g.vw[v];
            }
            fm_refine(g, side, eps);
            const long c = cut_of(g, side);
            if (best_cut < 0 || c < best_cut) {
                best_cut = c;
                best_side = side;
            }
        }
        return best_side;
    }
    std::vector<int> map;
    const Graph c = coarsen(g, map, rng);
    if (c.n() > n * 0.9) {  // matching stalled: refine from a random balanced start
        std::vector<char> side(n, 0);
        for (int v = 0; v < n; ++v) side[v] = static_cast<char>(v % 2);
        fm_refine(g, side, eps);
        return side;
    }
    const std::vector<char> cs = bisect_graph(c, eps, rng);
    std::vector<char> side(n);
    for (int v = 0; v < n; ++v) side[v] = cs[map[v]];
    fm_refine(g, side, eps);
    return side;
}

struct PartParams {
    double eps = 0.1;
    int cutoff = 16;
    GreedyParams gp;
};

int partition_tree(const Problem& pb, const Reduced& rd, const std::vector<std::vector<int>>& lab_holders,
                   const std::vector<int>& members, Tree& t, const PartParams& pp, std::mt19937_64& rng) {
    const int n = static_cast<int>(members.size());
    if (n <= pp.cutoff) {
        GreedyParams gp = pp.gp;
        gp.seed = rng();
        return greedy_subset(pb, rd, members, t, gp);
    }
    // local graph
    std::vector<int> local(rd.node.size(), -1);
    for (int i = 0; i < n; ++i) local[members[i]] = i;
    Graph g;
    g.vw.assign(n, 1);
    g.adj.assign(n, {});
    for (int i = 0; i < n; ++i) {
        auto& out = g.adj[i];
        rd.labels[members[i]].each([&](int l) {
            for (int h : lab_holders[l]) {
                const int j = local[h];
                if (j < 0 || j == i) continue;
                auto it = std::find_if(out.begin(), out.end(), [j](const std::pair<int, int>& e) { return e.first == j; });
                if (it == out.end()) out.push_back({j, 1});
                else ++it->second;
            }
        });
    }
    const std::vector<char> side = bisect_graph(g, pp.eps, rng);
    std::vector<int> A, B;
    for (int i = 0; i < n; ++i) (side[i] ? B : A).push_back(members[i]);
    if (A.empty() || B.empty()) {
        GreedyParams gp = pp.gp;
        gp.seed = rng();
        return greedy_subset(pb, rd, members, t, gp);
    }
    const int a = partition_tree(pb, rd, lab_holders, A, t, pp, rng);
    const int b = partition_tree(pb, rd, lab_holders, B, t, pp, rng);
    t.l.push_back(a);
    t.r.push_back(b);
    return static_cast<int>(t.l.size()) - 1;
}

// ---------------------------------------------------------------- slicing
// Adds sliced labels until the widest tensor fits; each pick is the label of a
// widest tensor that minimises the total (sliced) cost.
constexpr int kMaxIn = 8;       // inputs per reconfigured subtree (3^8 DP splits)
constexpr int kMaxInDeep = 10;  // the winner's final polish (3^10)
bool reconfigure_pass(const Problem& pb, Tree& t, const LSet& sliced, int n_sliced, double width,
                      int max_in = kMaxIn);

// One slicing step: the label of a widest tensor that minimises the total
// (sliced) cost.  Returns false when the widest tensor already fits.
bool slice_one(const Problem& pb, const Tree& t, LSet& sliced, int& n_sliced) {
    Eval e = evaluate(pb, t, sliced, n_sliced);
    if (e.max_size <= pb.width + 1e-9) return false;
    const int n = static_cast<int>(t.l.size());
    // candidates: labels of the widest tensors
    LSet cand(pb.n_labels);
    for (int v = 0; v < n; ++v)
        if (e.labels[v].count() + e.var[v] >= e.max_size - 1e-9)
            for (std::size_t k = 0; k < cand.w.size(); ++k) cand.w[k] |= e.labels[v].w[k];
    for (std::size_t k = 0; k < cand.w.size(); ++k) cand.w[k] &= ~pb.open.w[k];
    const std::vector<int> order = post_order(t);
    const double mult1 = std::ldexp(1.0, n_sliced + 1);
    int best = -1;
    double best_total = std::numeric_limits<double>::infinity();
    cand.each([&](int l) {
        double tot = 0;
        for (int v : order) {
            const int a = t.l[v], b = t.r[v];
            const bool in = e.labels[a].has(l) || e.labels[b].has(l);
            const bool dep = e.dep[v] || e.sub[v].has(l);
            tot += std::exp2(e.cost[v] - (in ? 1.0 : 0.0)) * (dep ? mult1 : 1.0);
        }
        if (tot < best_total) {
            best_total = tot;
            best = l;
        }
    });
    if (best < 0) throw ConfigError("scale planner: cannot slice below the memory budget (open legs too wide)");
    sliced.set(best);
    ++n_sliced;
    return true;
}

// Adds sliced labels until the widest tensor fits.
void slice_to_width(const Problem& pb, const Tree& t, LSet& sliced, int& n_sliced) {
    for (int guard = 0; guard < pb.n_labels; ++guard)
        if (!slice_one(pb, t, sliced, n_sliced)) return;
    throw ConfigError("scale planner: slicing did not converge");
}

// Slice-and-reconfigure from the unsliced tree: one label at a time, each
// followed by a reconfiguration pass that may not widen the tree, so the tree
// adapts to every cut before the next one is chosen.
void slice_and_reconfigure(const Problem& pb, Tree& t, LSet& sliced, int& n_sliced, int max_in) {
    sliced = LSet(pb.n_labels);
    n_sliced = 0;
    for (int guard = 0; guard < pb.n_labels; ++guard) {
        const double w = evaluate(pb, t, sliced, n_sliced).max_size;
        reconfigure_pass(pb, t, sliced, n_sliced, std::max(w, pb.width), max_in);
        if (!slice_one(pb, t, sliced, n_sliced)) return;
    }
    throw ConfigError("scale planner: slicing did not converge");
}

// ---------------------------------------------------------------- reconfiguration
// Re-contracts the subtree at v, cut at up to kMaxIn inputs, optimally by DP
// over input subsets.  Returns true if the subtree's cost dropped.

bool reconfigure_at(const Problem& pb, Tree& t, const Eval& e, int v, int n_sliced, std::vector<int>& free_ids,
                    double width, int max_in) {
    if (t.l[v] < 0) return false;
    // frontier: expand the widest internal node until kMaxIn inputs
    std::vector<int> in{t.l[v], t.r[v]}, inner{v};
    while (static_cast<int>(in.size()) < max_in) {
        int pick = -1;
        double ps = -1;
        for (std::size_t i = 0; i < in.size(); ++i) {
            const int x = in[i];
            if (t.l[x] < 0) continue;
            const double s = e.cost[x];
            if (s > ps) {
                ps = s;
                pick = static_cast<int>(i);
            }
        }
        if (pick < 0) break;
        const int x = in[pick];
        inner.push_back(x);
        in[pick] = t.l[x];
        in.push_back(t.r[x]);
    }
    const int k = static_cast<int>(in.size());
    if (k < 3) return false;
    // old cost of the inner steps
    const double mult = std::ldexp(1.0, n_sliced);
    double old_cost = 0;
    for (int x : inner) old_cost += std::exp2(e.cost[x]) * (e.dep[x] ? mult : 1.0);
    // local label index
    LSet all(pb.n_labels);
    for (int x : in)
        for (std::size_t w = 0; w < all.w.size(); ++w) all.w[w] |= e.labels[x].w[w];
    std::vector<int> glob;
    all.each([&](int l) { glob.push_back(l); });
    if (glob.size() > 256) return false;
    using B4 = std::array<std::uint64_t, 4>;
    auto pc = [](const B4& b) { return std::popcount(b[0]) + std::popcount(b[1]) + std::popcount(b[2]) + std::popcount(b[3]); };
    std::vector<B4> li(k, B4{0, 0, 0, 0});
    for (int i = 0; i < k; ++i)
        for (std::size_t j = 0; j < glob.size(); ++j)
            if (e.labels[in[i]].has(glob[j])) li[i][j >> 6] |= std::uint64_t{1} << (j & 63);
    const int full = (1 << k) - 1;
    std::vector<B4> L(full + 1, B4{0, 0, 0, 0});
    std::vector<int> outs(full + 1, 0), dep(full + 1, 0);
    // outs per input: variant bits are min(logM, outs); recover outs from var (exact below log_m)
    std::vector<int> in_outs(k);
    for (int i = 0; i < k; ++i) in_outs[i] = e.var[in[i]];
    for (int S = 1; S <= full; ++S) {
        const int i = std::countr_zero(static_cast<unsigned>(S));
        const int rest = S & (S - 1);
        for (int w = 0; w < 4; ++w) L[S][w] = L[rest][w] ^ li[i][w];
        outs[S] = outs[rest] + in_outs[i];
        dep[S] = dep[rest] || e.dep[in[i]];
    }
    const double inf = std::numeric_limits<double>::infinity();
    std::vector<double> best(full + 1, inf);
    std::vector<int> split(full + 1, 0);
    for (int i = 0; i < k; ++i) best[1 << i] = 0;
    for (int S = 1; S <= full; ++S) {
        if (std::popcount(static_cast<unsigned>(S)) < 2) continue;
        const double var = vbits(pb, outs[S]);
        const double size = pc(L[S]) + var;
        if (S != full && size > width + 1e-9) continue;
        const double w = dep[S] ? mult : 1.0;
        const int low = S & -S;
        // A contains the lowest input (each unordered split once)
        for (int A = (S - 1) & S; A > 0; A = (A - 1) & S) {
            if (!(A & low)) continue;
            const int Bm = S ^ A;
            if (best[A] == inf || best[Bm] == inf) continue;
            B4 u;
            for (int q = 0; q < 4; ++q) u[q] = L[A][q] | L[Bm][q];
            const double c = best[A] + best[Bm] +
                             step_cost(pc(u) + var + 3.0, pc(L[A]) + vbits(pb, outs[A]), pc(L[Bm]) + vbits(pb, outs[Bm]),
                                       size) * w;
            if (c < best[S]) {
                best[S] = c;
                split[S] = A;
            }
        }
    }
    if (!(best[full] < old_cost * (1 - 1e-9))) return false;
    // rebuild: reuse the inner node ids (v stays the subtree root)
    std::vector<int> ids(inner.begin() + 1, inner.end());
    std::function<int(int, bool)> build = [&](int S, bool is_root) -> int {
        if (std::popcount(static_cast<unsigned>(S)) == 1) return in[std::countr_zero(static_cast<unsigned>(S))];
        const int A = split[S];
        const int a = build(A, false), b = build(S ^ A, false);
        int id;
        if (is_root) id = v;
        else if (!ids.empty()) {
            id = ids.back();
            ids.pop_back();
        } else {
            id = free_ids.back();
            free_ids.pop_back();
        }
        t.l[id] = a;
        t.r[id] = b;
        return id;
    };
    build(full, true);
    return true;
}

// One pass over every internal node, costliest steps first (internal ids are
// arbitrary here; emit() numbers the steps in post-order).
bool reconfigure_pass(const Problem& pb, Tree& t, const LSet& sliced, int n_sliced, double width, int max_in) {
    bool any = false;
    Eval e = evaluate(pb, t, sliced, n_sliced);
    std::vector<int> order = post_order(t);
    std::sort(order.begin(), order.end(), [&](int a, int b) { return e.cost[a] > e.cost[b]; });
    std::vector<int> free_ids;
    for (int v : order) {
        if (reconfigure_at(pb, t, e, v, n_sliced, free_ids, width < 0 ? pb.width : width, max_in)) {
            any = true;
            e = evaluate(pb, t, sliced, n_sliced);  // the subtree's node ids now hold new contractions
        }
    }
    return any;
}

// ---------------------------------------------------------------- plan output
ContractionPlan emit(const Problem& pb, const Tree& t, const TensorNetwork& net, const LSet& sliced_set,
                     const std::vector<Label>& sliced, const std::vector<Label>& broken,
                     const std::vector<Label>& fixed, std::uint64_t budget) {
    ContractionPlan plan;
    plan.sliced = sliced;
    plan.broken = broken;
    plan.fixed_outputs = fixed;
    plan.memory_budget_bytes = budget;
    (void)net;
    const int n = static_cast<int>(t.l.size());
    std::vector<LSet> lab(n, LSet(pb.n_labels));
    std::vector<int> id(n, -1);
    std::vector<double> bytes(n, 0);
    constexpr double kSat = 1.8446744073709552e19;
    auto sat = [&](double x) { return x >= kSat ? ~std::uint64_t{0} : static_cast<std::uint64_t>(x); };
    double live = 0, peak = 0, flops = 0, traffic = 0;
    for (int i = 0; i < pb.n_leaves; ++i) {
        lab[i] = pb.leaf[i];
        for (std::size_t k = 0; k < lab[i].w.size(); ++k) lab[i].w[k] &= ~sliced_set.w[k];
        id[i] = i;
        bytes[i] = 16.0 * std::exp2(lab[i].count());
        live += bytes[i];
    }
    peak = live;
    int next = pb.n_leaves;
    for (int v : post_order(t)) {
        const int a = t.l[v], b = t.r[v];
        const int shared = lab[a].and_count(lab[b]);
        lab[v] = lab[a];
        lab[v].xor_in(lab[b]);
        const int rr = lab[v].count();
        bytes[v] = 16.0 * std::exp2(rr);
        const double f = 8.0 * std::exp2(rr + shared);
        const double io = bytes[a] + bytes[b] + bytes[v];
        peak = std::max(peak, live + io);
        flops += f;
        traffic += io;
        live = std::max(0.0, live + bytes[v] - bytes[a] - bytes[b]);
        PlanStep s;
        s.lhs = id[a];
        s.rhs = id[b];
        s.result = next;
        id[v] = next++;
        s.summed = static_cast<std::uint64_t>(shared);
        s.flops = sat(f);
        s.result_bytes = sat(bytes[v]);
        lab[v].each([&s](int l) { s.result_labels.push_back(l); });
        plan.steps.push_back(std::move(s));
    }
    plan.flops_per_slice = sat(flops);
    plan.traffic_bytes_per_slice = sat(traffic);
    plan.peak_bytes = sat(peak);
    return plan;
}

}  // namespace

ContractionPlan find_contraction_path_scale(const TensorNetwork& network, std::uint64_t memory_budget_bytes,
                                            SearchEffort effort, std::uint64_t seed,
                                            const std::vector<Label>& broken, const ScalePlannerOptions& opt,
                                            ScalePlanReport* report) {
    const auto t_start = std::chrono::steady_clock::now();
    Problem pb;
    pb.n_labels = static_cast<int>(network.label_names.size());
    pb.n_leaves = static_cast<int>(network.tensors.size());
    if (pb.n_leaves < 1) throw ConfigError("network has no tensors");
    pb.log_m = opt.n_groups > 1 ? std::ceil(std::log2(static_cast<double>(opt.n_groups))) : 0.0;
    if (memory_budget_bytes < 64) throw ConfigError("memory budget is infeasible");
    pb.width = std::floor(std::log2(static_cast<double>(memory_budget_bytes) / 64.0));  // 16 B/amp, budget/4
    LSet removed(pb.n_labels);
    std::vector<Label> fixed;
    for (Label l : broken) removed.set(l);
    std::vector<char> is_fixed(pb.n_labels, 0);
    for (Label l : network.output_labels)
        if (!network.is_open(l)) {
            removed.set(l);
            fixed.push_back(l);
            is_fixed[l] = 1;
        }
    pb.open = LSet(pb.n_labels);
    for (Label l : network.open_labels) pb.open.set(l);
    pb.leaf.assign(pb.n_leaves, LSet(pb.n_labels));
    pb.leaf_out.assign(pb.n_leaves, 0);
    for (int i = 0; i < pb.n_leaves; ++i) {
        for (Label l : network.tensors[i].labels) {
            if (l < 0 || l >= pb.n_labels) throw ConfigError("tensor label out of range");
            if (is_fixed[l]) ++pb.leaf_out[i];
            if (!removed.has(l)) pb.leaf[i].set(l);
        }
        if (pb.leaf[i].count() + vbits(pb, pb.leaf_out[i]) > pb.width)
            throw ConfigError("memory budget " + std::to_string(memory_budget_bytes) +
                              " B is infeasible: smaller than a single tensor");
    }
    const int trials = opt.trials > 0 ? opt.trials
                                      : (effort == SearchEffort::Low ? 256 : effort == SearchEffort::Medium ? 1024 : 4096);
    int threads = opt.threads > 0 ? opt.threads : static_cast<int>(std::thread::hardware_concurrency());
    threads = std::max(1, std::min(threads, trials));
    const bool debug = getenv("RCSG_PLAN_DEBUG") != nullptr;
    // RCSG_PLAN_REFINE: size of the reconfiguration pool (search experiments)
    const int refine = getenv("RCSG_PLAN_REFINE") ? atoi(getenv("RCSG_PLAN_REFINE")) : opt.refine;
    // RCSG_PLAN_SEED: an independent trial stream (offline plan searches; plan files)
    if (const char* s = getenv("RCSG_PLAN_SEED")) seed ^= std::strtoull(s, nullptr, 0) * 0x94d049bb133111ebull;
    std::mutex debug_mu;
    struct Result {
        double total = std::numeric_limits<double>::infinity();
        Tree tree;
        LSet sliced;
        int n_sliced = 0;
        int trial = -1;
    };
    int reduced_tensors = 0;
    // One search phase: trees are built on the network with `pre` labels removed
    // (phase 1: none; phase 2: the best phase-1 slice set, so the partitions see
    // the sliced network), sliced further to the width limit starting from
    // `pre`, and the best few are refined by reconfiguration.
    auto phase = [&](const LSet& pre, int n_pre, int phase_id) {
        Problem tb = pb;  // tree-building view: pre-sliced labels cut
        for (auto& lf : tb.leaf)
            for (std::size_t k = 0; k < lf.w.size(); ++k) lf.w[k] &= ~pre.w[k];
        Tree base;
        base.l.assign(pb.n_leaves, -1);
        base.r.assign(pb.n_leaves, -1);
        const Reduced rd = simplify(tb, base);
        reduced_tensors = static_cast<int>(rd.node.size());
        std::vector<std::vector<int>> lab_holders(pb.n_labels);
        for (int i = 0; i < static_cast<int>(rd.node.size()); ++i)
            rd.labels[i].each([&](int l) { lab_holders[l].push_back(i); });
        const int keep = std::max(1, refine);
        std::vector<std::vector<Result>> tops(threads);  // per worker: its `keep` best trees
        std::atomic<int> next_trial{0};
        auto worker = [&](int w) {
            for (int tr; (tr = next_trial.fetch_add(1)) < trials;) {
                std::mt19937_64 rng(seed * 0x9e3779b97f4a7c15ull + static_cast<std::uint64_t>(tr) * 0xd1b54a32d192ed03ull +
                                    1 + static_cast<std::uint64_t>(phase_id) * 0x632be59bd9b4e019ull);
                std::uniform_real_distribution<double> U(0.0, 1.0);
                GreedyParams gp;
                if (tr == 0) {  // one plain greedy (alpha 1, no noise)
                    gp.alpha = 1.0;
                    gp.temp = 0.0;
                } else {
                    gp.alpha = 2.0 * U(rng);
                    gp.temp = std::exp(std::log(1e-3) + U(rng) * (std::log(1.0) - std::log(1e-3)));
                }
                gp.seed = rng();
                Tree t = base;
                if (tr % 4 == 0) {  // a quarter of the trials: randomized greedy on the whole network
                    greedy(tb, rd, t, gp);
                } else {            // the rest: recursive multilevel bisection, greedy below the cutoff
                    PartParams pp;
                    pp.eps = std::exp(std::log(0.01) + U(rng) * (std::log(0.99) - std::log(0.01)));
                    pp.cutoff = 4 + static_cast<int>(U(rng) * 36);
                    pp.gp = gp;
                    pp.gp.temp *= 0.1;
                    std::vector<int> all(rd.node.size());
                    std::iota(all.begin(), all.end(), 0);
                    t.root = partition_tree(tb, rd, lab_holders, all, t, pp, rng);
                }
                LSet sl = pre;
                int ns = n_pre;
                try {
                    slice_to_width(pb, t, sl, ns);
                } catch (const ConfigError&) {
                    continue;
                }
                const double tot = evaluate(pb, t, sl, ns).total;
                if (debug) {
                    std::lock_guard<std::mutex> lk(debug_mu);
                    fprintf(stderr, "[plan] phase %d trial %d %s log2 total %.2f sliced %d\n", phase_id, tr,
                            tr % 4 == 0 ? "greedy" : "partition", std::log2(tot), ns);
                }
                auto& top = tops[w];
                if (static_cast<int>(top.size()) < keep || tot < top.back().total) {
                    top.push_back(Result{tot, std::move(t), sl, ns, tr});
                    std::sort(top.begin(), top.end(), [](const Result& a, const Result& b) { return a.total < b.total; });
                    if (static_cast<int>(top.size()) > keep) top.pop_back();
                }
            }
        };
        {
            std::vector<std::thread> pool;
            for (int w = 1; w < threads; ++w) pool.emplace_back(worker, w);
            worker(0);
            for (auto& th : pool) th.join();
        }
        std::vector<Result> best_of;
        for (auto& top : tops)
            for (auto& r : top) best_of.push_back(std::move(r));
        if (best_of.empty()) best_of.resize(1);
        std::sort(best_of.begin(), best_of.end(), [](const Result& a, const Result& b) {
            return a.total < b.total || (a.total == b.total && a.trial < b.trial);
        });
        // reconfigure the best few trees (in parallel), re-slicing as needed
        const int n_refine = std::min<int>(std::max(1, refine), static_cast<int>(best_of.size()));
        std::vector<std::thread> pool;
        for (int i = 0; i < n_refine; ++i)
            pool.emplace_back([&, i] {
                Result& r = best_of[i];
                if (r.trial < 0) return;
                if (i < 16 && r.n_sliced > 0) {  // the best few also try slice-and-reconfigure
                    Result alt = r;
                    try {
                        slice_and_reconfigure(pb, alt.tree, alt.sliced, alt.n_sliced, kMaxIn);
                        alt.total = evaluate(pb, alt.tree, alt.sliced, alt.n_sliced).total;
                        if (alt.total < r.total) r = std::move(alt);
                    } catch (const ConfigError&) {
                    }
                }
                for (int round = 0; round < 8; ++round) {
                    bool changed = false;
                    for (int pass = 0; pass < 6 && reconfigure_pass(pb, r.tree, r.sliced, r.n_sliced, -1); ++pass)
                        changed = true;
                    // try dropping sliced labels the reconfigured tree no longer needs
                    std::vector<int> sl;
                    r.sliced.each([&](int l) { sl.push_back(l); });
                    for (int l : sl) {
                        LSet trial = r.sliced;
                        trial.reset(l);
                        const Eval e = evaluate(pb, r.tree, trial, r.n_sliced - 1);
                        if (e.max_size <= pb.width + 1e-9) {
                            r.sliced = trial;
                            --r.n_sliced;
                            changed = true;
                        }
                    }
                    if (!changed) break;
                }
                const double before = r.total;
                r.total = evaluate(pb, r.tree, r.sliced, r.n_sliced).total;
                if (debug) {
                    std::lock_guard<std::mutex> lk(debug_mu);
                    fprintf(stderr, "[plan] phase %d refine trial %d: log2 total %.2f -> %.2f sliced %d\n", phase_id,
                            r.trial, std::log2(before), std::log2(r.total), r.n_sliced);
                }
            });
        for (auto& th : pool) th.join();
        std::sort(best_of.begin(), best_of.begin() + n_refine, [](const Result& a, const Result& b) {
            return a.total < b.total || (a.total == b.total && a.trial < b.trial);
        });
        return best_of[0];
    };
    Result best = phase(LSet(pb.n_labels), 0, 0);
    if (!(best.total < std::numeric_limits<double>::infinity()))
        throw ConfigError("scale planner: no trial fits the memory budget");
    // final polish of the winner: deeper subtrees (10 inputs), then drop unneeded slices
    for (int round = 0; round < 4; ++round) {
        bool changed = false;
        for (int pass = 0; pass < 4 && reconfigure_pass(pb, best.tree, best.sliced, best.n_sliced, -1, kMaxInDeep);
             ++pass)
            changed = true;
        std::vector<int> sl;
        best.sliced.each([&](int l) { sl.push_back(l); });
        for (int l : sl) {
            LSet trial = best.sliced;
            trial.reset(l);
            if (evaluate(pb, best.tree, trial, best.n_sliced - 1).max_size <= pb.width + 1e-9) {
                best.sliced = trial;
                --best.n_sliced;
                changed = true;
            }
        }
        if (!changed) break;
    }
    best.total = evaluate(pb, best.tree, best.sliced, best.n_sliced).total;
    // phase 2 (sliced plans): search again on the network with the phase-1 slice set cut
    if (best.n_sliced > 0 && opt.phases > 1) {
        Result second = phase(best.sliced, best.n_sliced, 1);
        if (second.total < best.total) {
            second.trial += trials;  // report phase-2 winners after phase-1 trial ids
            best = std::move(second);
        }
    }
    const Result& win = best;
    // sliced labels in ascending label order (slice bit b <-> sliced[b])
    std::vector<Label> sliced;
    win.sliced.each([&](int l) { sliced.push_back(l); });
    ContractionPlan plan = emit(pb, win.tree, network, win.sliced, sliced, broken, fixed, memory_budget_bytes);
    if (report) {
        const Eval e = evaluate(pb, win.tree, win.sliced, win.n_sliced);
        report->log2_total_flops = std::log2(e.flops);
        if (debug) {  // the winner under the roofline time model (ridge 128 FLOP/B)
            double t = 0, mem = 0;
            for (int v = pb.n_leaves; v < static_cast<int>(win.tree.l.size()); ++v) {
                if (win.tree.l[v] < 0) continue;
                const int a = win.tree.l[v], b = win.tree.r[v];
                const double fl = e.labels[a].union_count(e.labels[b]) + e.var[v] + 3.0;
                const double c = step_cost(fl, e.labels[a].count() + e.var[a], e.labels[b].count() + e.var[b],
                                           e.labels[v].count() + e.var[v], 128.0);
                const double w = e.dep[v] ? std::exp2(win.n_sliced) : 1.0;
                t += c * w;
                if (c > std::exp2(fl)) mem += c * w;
            }
            fprintf(stderr, "[plan] winner: log2 flops %.2f, log2 time-model cost %.2f (memory-bound share %.2f)\n",
                    std::log2(e.flops), std::log2(t), mem / t);
        }
        double per_slice = 0, once = 0;
        for (int v = pb.n_leaves; v < static_cast<int>(win.tree.l.size()); ++v) {
            if (win.tree.l[v] < 0) continue;
            const int a = win.tree.l[v], b = win.tree.r[v];
            (e.dep[v] ? per_slice : once) += std::exp2(e.labels[a].union_count(e.labels[b]) + e.var[v] + 3.0);
        }
        report->log2_flops_per_slice_batched = std::log2(per_slice);
        report->log2_flops_once_batched = once > 0 ? std::log2(once) : -1;
        report->log2_max_size = e.max_size;
        report->n_sliced = win.n_sliced;
        report->trials = trials;
        report->winning_trial = win.trial;
        report->threads = threads;
        report->reduced_tensors = reduced_tensors;
        report->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    }
    return plan;
}

namespace {
PlannerKind g_planner = PlannerKind::Auto;
ScalePlannerOptions g_scale_options;
}  // namespace

void set_planner(PlannerKind kind, const ScalePlannerOptions& options) {
    g_planner = kind;
    g_scale_options = options;
}
PlannerKind get_planner() { return g_planner; }

// find_contraction_path (contraction_plan.hpp:67-70): the reference algorithm
// (bit-identical plans) wherever it works; the scale planner where its costs
// overflow or its slicing stalls (PlannerKind::Auto), or when selected.
ContractionPlan find_contraction_path(const TensorNetwork& network, std::uint64_t memory_budget_bytes,
                                      SearchEffort effort, std::uint64_t seed, const std::vector<Label>& broken) {
    switch (g_planner) {
        case PlannerKind::Reference:
            return find_contraction_path_reference(network, memory_budget_bytes, effort, seed, broken);
        case PlannerKind::Scale:
            return find_contraction_path_scale(network, memory_budget_bytes, effort, seed, broken, g_scale_options);
        case PlannerKind::Auto:
        default:
            break;
    }
    if (reference_planner_overflows(network, broken))
        return find_contraction_path_scale(network, memory_budget_bytes, effort, seed, broken, g_scale_options);
    try {
        return find_contraction_path_reference(network, memory_budget_bytes, effort, seed, broken);
    } catch (const ConfigError& e) {
        if (std::string(e.what()).rfind("cannot slice below memory budget", 0) != 0) throw;
        return find_contraction_path_scale(network, memory_budget_bytes, effort, seed, broken, g_scale_options);
    }
}

}  // namespace rcs
