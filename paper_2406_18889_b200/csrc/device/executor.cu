// Step-program executor; see executor.hpp for the design.
#include <algorithm>
#include <array>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <iterator>
#include <numeric>
#include <type_traits>

#include "executor.hpp"

namespace rcsg {

#define CUDA_OK(x)                                                                      \
    do {                                                                                \
        cudaError_t e_ = (x);                                                           \
        if (e_ != cudaSuccess)                                                          \
            throw Failure{RCSG_ERR_DEVICE, std::string("CUDA: ") + cudaGetErrorString(e_) + \
                                               " at " #x};                              \
    } while (0)

// run BODY with S = the storage type of precision PREC
#define RCSG_DISPATCH(PREC, BODY)              \
    do {                                       \
        if ((PREC) == RCSG_PREC_F64) {         \
            using S = double;                  \
            BODY;                              \
        } else if ((PREC) == RCSG_PREC_BF16) { \
            using S = bf16;                    \
            BODY;                              \
        } else if ((PREC) == RCSG_PREC_F16) {  \
            using S = f16;                     \
            BODY;                              \
        } else {                               \
            using S = float;                   \
            BODY;                              \
        }                                      \
    } while (0)

namespace {

constexpr int64_t kAlign = 64;  // elements; keeps every plane 256-B aligned

int64_t align_up(int64_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

// First-fit allocator simulation (offsets in elements).
struct FirstFit {
    std::map<int64_t, int64_t> free_;  // offset -> size
    int64_t top = 0, peak = 0;
    int64_t alloc(int64_t size) {
        size = align_up(std::max<int64_t>(size, 1));
        for (auto it = free_.begin(); it != free_.end(); ++it)
            if (it->second >= size) {
                const int64_t off = it->first, rem = it->second - size;
                free_.erase(it);
                if (rem) free_[off + size] = rem;
                return off;
            }
        // extend the top (merging a trailing free block)
        int64_t off = top;
        if (!free_.empty()) {
            auto last = std::prev(free_.end());
            if (last->first + last->second == top) {
                off = last->first;
                free_.erase(last);
            }
        }
        top = off + size;
        peak = std::max(peak, top);
        return off;
    }
    void release(int64_t off, int64_t size) {
        size = align_up(std::max<int64_t>(size, 1));
        auto it = free_.emplace(off, size).first;
        auto nx = std::next(it);
        if (nx != free_.end() && it->first + it->second == nx->first) {
            it->second += nx->second;
            free_.erase(nx);
        }
        if (it != free_.begin()) {
            auto pv = std::prev(it);
            if (pv->first + pv->second == it->first) {
                pv->second += it->second;
                free_.erase(it);
                it = pv;
            }
        }
        if (it->first + it->second == top) {
            top = it->first;
            free_.erase(it);
        }
    }
};

int64_t pos_in(const std::vector<int>& v, int x) {
    for (size_t i = 0; i < v.size(); ++i)
        if (v[i] == x) return static_cast<int64_t>(i);
    return -1;
}

// src_bit for permuting layout `from` into layout `to` (both MSB-first label lists)
void permute_bits(const std::vector<int>& from, const std::vector<int>& to, std::vector<int>& src_bit) {
    const int r = static_cast<int>(to.size());
    src_bit.assign(r, 0);
    for (int q = 0; q < r; ++q) {
        const int label = to[r - 1 - q];
        src_bit[q] = r - 1 - static_cast<int>(pos_in(from, label));
    }
}

// ---- batch-aware reassociation of the contraction tree -------------------
// The reference plans one group's network (var legs projected).  With a group
// batch, a node's cost is multiplied by its variant count (distinct
// projections of the batch's prefixes onto the output legs in its subtree),
// so the single-group optimum pushes group-dependent work into the big stem
// steps.  Local rotations fix that: for P = (Z, W) with Z = (X, Y), try
// P = (X, (Y, W)) and P = (Y, (X, W)); keep a rotation when the modelled time
// of the two steps drops.  P's labels and subtree are unchanged, so the
// result is the same tensor (up to rounding); slices, configurations and the
// canonical output order are untouched.  SURVEY §8f row 2 ("group batching as
// a plan transform", the paper's sparse-state stage).
struct TreeNode {
    std::vector<int> labels;  // free labels, sorted
    uint64_t mask = 0;        // group-code bits in the subtree
    int level = 0;            // 0 constant, 1 per pass, 2 per group
    int a = -1, b = -1;       // children (internal nodes)
};

struct TreeCost {
    const std::vector<uint64_t>& groups;
    double pf, bw, elem, lat;
    std::map<uint64_t, double> nv_cache;
    double nvar(uint64_t mask) {
        if (!mask) return 1.0;
        auto it = nv_cache.find(mask);
        if (it != nv_cache.end()) return it->second;
        std::vector<uint64_t> v;
        v.reserve(groups.size());
        for (uint64_t g : groups) v.push_back(g & mask);
        std::sort(v.begin(), v.end());
        const double n = static_cast<double>(std::unique(v.begin(), v.end()) - v.begin());
        nv_cache[mask] = n;
        return n;
    }
    // modelled seconds of one contraction step (the executor's GEMM modes)
    double step(const TreeNode& x, const TreeNode& y) {
        std::vector<int> sh;
        std::set_intersection(x.labels.begin(), x.labels.end(), y.labels.begin(), y.labels.end(),
                              std::back_inserter(sh));
        const double la = std::ldexp(1.0, static_cast<int>(x.labels.size()));
        const double lb = std::ldexp(1.0, static_cast<int>(y.labels.size()));
        const double lz = std::ldexp(1.0, static_cast<int>(x.labels.size() + y.labels.size() - 2 * sh.size()));
        const double un = std::ldexp(1.0, static_cast<int>(x.labels.size() + y.labels.size() - sh.size()));
        const double va = nvar(x.mask), vb = nvar(y.mask), vz = nvar(x.mask | y.mask);
        double mult, rd;
        if (x.mask && y.mask) {
            mult = vz;
            const uint64_t hx = x.mask, hy = y.mask;
            const bool separable = __builtin_ctzll(hx) > 63 - __builtin_clzll(hy) ||
                                   __builtin_ctzll(hy) > 63 - __builtin_clzll(hx);
            if (separable && vz == va * vb) rd = va * la + vb * lb;  // product: one GEMM, variants in M and N
            else rd = vz * (la + lb);                                // gathered batch: one GEMM per variant
        } else {  // the varying operand's variants fold into M
            mult = std::max(va, vb);
            rd = va * la + vb * lb;
        }
        const double t = std::max(8.0 * un * mult / pf, 2.0 * elem * (rd + vz * lz) / bw) + lat;
        // level-0 steps run once per call, not per pass
        return std::max(x.level, y.level) == 0 ? 0.01 * t : t;
    }
};

void combine(std::vector<TreeNode>& t, int r) {
    TreeNode& z = t[r];
    const TreeNode &x = t[z.a], &y = t[z.b];
    z.labels.clear();
    std::set_symmetric_difference(x.labels.begin(), x.labels.end(), y.labels.begin(), y.labels.end(),
                                  std::back_inserter(z.labels));
    z.mask = x.mask | y.mask;
    z.level = std::max(x.level, y.level);
}

// steps: (a, b, r) triples, rewritten in place; origin[i]: plan index of step i.
// Returns the number of rotations applied.
int reassociate(std::vector<TreeNode>& t, std::vector<int32_t>& steps, std::vector<int32_t>& origin,
                TreeCost& cost, double max_elems) {
    const int n_steps = static_cast<int>(steps.size() / 3);
    std::vector<int> pos(t.size(), -1);  // node -> step producing it
    auto reindex = [&] {
        for (int i = 0; i < n_steps; ++i) pos[steps[3 * i + 2]] = i;
    };
    reindex();
    int rotations = 0;
    for (int round = 0; round < 64; ++round) {
        bool improved = false;
        for (int i = 0; i < n_steps; ++i) {
            const int P = steps[3 * i + 2];
            for (int zi = 0; zi < 2; ++zi) {
                const int Z = zi == 0 ? t[P].a : t[P].b;
                const int W = zi == 0 ? t[P].b : t[P].a;
                if (pos[Z] < 0) continue;  // a leaf
                const int X = t[Z].a, Y = t[Z].b;
                const double base = cost.step(t[X], t[Y]) + cost.step(t[Z], t[W]);
                double best = base * 0.999;
                int bu = -1, bv = -1;
                for (int o = 0; o < 2; ++o) {
                    const int u = o == 0 ? X : Y, v = o == 0 ? Y : X;
                    std::vector<int> sh;
                    std::set_intersection(t[v].labels.begin(), t[v].labels.end(), t[W].labels.begin(),
                                          t[W].labels.end(), std::back_inserter(sh));
                    if (sh.empty() && !(t[v].mask && t[W].mask)) continue;
                    TreeNode z2;
                    z2.a = v;
                    z2.b = W;
                    std::set_symmetric_difference(t[v].labels.begin(), t[v].labels.end(), t[W].labels.begin(),
                                                  t[W].labels.end(), std::back_inserter(z2.labels));
                    z2.mask = t[v].mask | t[W].mask;
                    z2.level = std::max(t[v].level, t[W].level);
                    if (z2.labels.size() > static_cast<size_t>(kMaxRank) ||
                        cost.nvar(z2.mask) * std::ldexp(1.0, static_cast<int>(z2.labels.size())) > max_elems)
                        continue;
                    const double c = cost.step(t[v], t[W]) + cost.step(t[u], z2);
                    if (c < best) {
                        best = c;
                        bu = u;
                        bv = v;
                    }
                }
                if (bu < 0) continue;
                // apply: Z = (bv, W) computed right before P; P = (bu, Z)
                t[Z].a = bv;
                t[Z].b = W;
                combine(t, Z);
                t[P].a = bu;
                t[P].b = Z;
                const int zs = pos[Z];
                const int32_t zo = origin[zs];
                steps.erase(steps.begin() + 3 * zs, steps.begin() + 3 * zs + 3);
                origin.erase(origin.begin() + zs);
                const int ps = pos[P] - 1;  // P's step moved up by one
                const int32_t tri[3] = {bv, W, Z};
                steps.insert(steps.begin() + 3 * ps, tri, tri + 3);
                origin.insert(origin.begin() + ps, zo);
                steps[3 * (ps + 1)] = bu;
                steps[3 * (ps + 1) + 1] = Z;
                reindex();
                ++rotations;
                improved = true;
                break;
            }
        }
        if (!improved) break;
    }
    return rotations;
}

}  // namespace

Program::Program(const rcsg_network_desc& net, const rcsg_plan_desc& plan,
                 const std::vector<LabelRole>& roles, int precision, uint64_t mem_budget)
    : precision_(precision), mem_budget_(mem_budget), roles_(roles) {
    if (precision < RCSG_PREC_F64 || precision > RCSG_PREC_F16)
        throw Failure{RCSG_ERR_CONFIG, "unknown precision"};
    elem_bytes_ = precision == RCSG_PREC_F64 ? 8 : (precision >= RCSG_PREC_BF16 ? 2 : 4);
    build_nodes(net, plan);
    build_steps();
    node_exp_.assign(nodes_.size(), 0);
    // keep the inputs: the first run may reassociate the tree (retree) and the
    // fp16 mode builds its calibration program from them
    calib_net_ = net;
    calib_plan_ = plan;
    c_rank_.assign(net.leaf_rank, net.leaf_rank + net.n_leaves);
    int64_t nl = 0;
    for (int i = 0; i < net.n_leaves; ++i) nl += net.leaf_rank[i];
    c_labels_.assign(net.leaf_labels, net.leaf_labels + nl);
    c_out_.assign(net.output_labels, net.output_labels + net.n_qubits);
    c_openl_.assign(net.open_labels, net.open_labels + net.n_open);
    c_openq_.assign(net.open_qubits, net.open_qubits + net.n_open);
    c_steps_.assign(plan.steps, plan.steps + 3 * plan.n_steps);
    c_sliced_.assign(plan.sliced, plan.sliced + plan.n_sliced);
    c_broken_.assign(plan.broken, plan.broken + plan.n_broken);
    c_fixed_.assign(plan.fixed_outputs, plan.fixed_outputs + plan.n_fixed);
    CUDA_OK(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    ls_ = stream_;
    // leaf data + pass sources + canonical map
    CUDA_OK(cudaMalloc(&d_leaf_data_, std::max<size_t>(leaf_data_.size(), 2) * sizeof(double)));
    CUDA_OK(cudaMemcpy(d_leaf_data_, leaf_data_.data(), leaf_data_.size() * sizeof(double),
                       cudaMemcpyHostToDevice));
    std::vector<PassSrc> src(roles_.size());
    for (size_t l = 0; l < roles_.size(); ++l) src[l] = roles_[l].src;
    CUDA_OK(cudaMalloc(&d_pass_src_, std::max<size_t>(src.size(), 1) * sizeof(PassSrc)));
    CUDA_OK(cudaMemcpy(d_pass_src_, src.data(), src.size() * sizeof(PassSrc), cudaMemcpyHostToDevice));
    CUDA_OK(cudaMalloc(&d_state_, sizeof(PassState)));
    CUDA_OK(cudaMemset(d_state_, 0, sizeof(PassState)));
    CUDA_OK(cudaMalloc(&d_canon_, std::max<size_t>(root_canon_src_.size(), 1) * sizeof(int32_t)));
    CUDA_OK(cudaMemcpy(d_canon_, root_canon_src_.data(), root_canon_src_.size() * sizeof(int32_t),
                       cudaMemcpyHostToDevice));
    CUDA_OK(cudaMalloc(&d_fault_, sizeof(int32_t)));
}

Program::~Program() {
    free_chunks();
    cudaFree(arena_);
    cudaFree(d_leaf_data_);
    cudaFree(d_pass_src_);
    cudaFree(d_state_);
    cudaFree(d_canon_);
    cudaFree(d_fault_);
    cudaFree(d_part_);
    cudaFree(d_res_);
    cudaFree(d_comp_);
    for (auto* p : d_static_jobs_) cudaFree(p);
    for (cudaEvent_t e : ev_pool_) cudaEventDestroy(e);
    if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
    free_tasks();
    for (void* t : tab_mem_) cudaFree(t);
    cudaFree(d_tab_jobs_);
    for (cudaEvent_t e : lane_ev_) cudaEventDestroy(e);
    for (cudaStream_t l : lanes_) {
        release_workspace(l);
        cudaStreamDestroy(l);
    }
    if (stream_) {
        release_workspace(stream_);
        cudaStreamDestroy(stream_);
    }
}

void Program::build_nodes(const rcsg_network_desc& net, const rcsg_plan_desc& plan) {
    n_leaves_ = net.n_leaves;
    const int n_nodes = net.n_leaves + plan.n_steps;
    if (net.n_leaves < 1) throw Failure{RCSG_ERR_CONFIG, "network has no tensors"};
    if (static_cast<int>(roles_.size()) != net.n_labels)
        throw Failure{RCSG_ERR_CONFIG, "label role table does not match the network"};
    nodes_.assign(n_nodes, NodeInfo{});
    canon_qubit_.assign(net.n_labels, -1);
    for (int j = 0; j < net.n_open; ++j) canon_qubit_[net.open_labels[j]] = net.open_qubits[j];
    // leaves: project away pinned labels (reference project_leaf keeps free labels in order)
    int64_t lo = 0, doff = 0;
    for (int i = 0; i < net.n_leaves; ++i) {
        NodeInfo& nd = nodes_[i];
        nd.is_leaf = true;
        nd.rank0 = net.leaf_rank[i];
        if (nd.rank0 > kMaxLeafRank) throw Failure{RCSG_ERR_CONFIG, "leaf tensor rank above 8 is unsupported"};
        nd.data_off = doff;
        bool pass = false;
        for (int p = 0; p < nd.rank0; ++p) {
            const int l = net.leaf_labels[lo + p];
            if (l < 0 || l >= net.n_labels) throw Failure{RCSG_ERR_CONFIG, "leaf label out of range"};
            nd.labels0.push_back(l);
            const LabelRole& rl = roles_[l];
            if (rl.role == kFree) nd.labels.push_back(l);
            else if (rl.role == kPass) {
                pass = true;
                if (rl.src.kind == 1) nd.slice_mask |= uint64_t{1} << rl.src.bit;
                if (rl.src.kind == 2) nd.cfg_dep = true;
            } else nd.var_mask |= uint64_t{1} << rl.var_bit;
        }
        nd.level = nd.var_mask ? 2 : (pass ? 1 : 0);
        nd.pass_dep = pass;
        nd.payload = int64_t{1} << nd.labels.size();
        lo += nd.rank0;
        doff += int64_t{1} << nd.rank0;
    }
    leaf_data_.assign(net.leaf_data, net.leaf_data + 2 * doff);
    // internal nodes: result of each step (post-order)
    std::vector<char> made(n_nodes, 0), used(n_nodes, 0);
    for (int i = 0; i < net.n_leaves; ++i) made[i] = 1;
    steps_.clear();
    plan_flops_ = 0;
    for (int s = 0; s < plan.n_steps; ++s) {
        const int a = plan.steps[3 * s], b = plan.steps[3 * s + 1], r = plan.steps[3 * s + 2];
        if (a < 0 || b < 0 || r < 0 || a >= n_nodes || b >= n_nodes || r >= n_nodes || a == b ||
            !made[a] || !made[b] || used[a] || used[b] || made[r])
            throw Failure{RCSG_ERR_CONFIG, "malformed contraction plan at step " + std::to_string(s)};
        used[a] = used[b] = 1;
        made[r] = 1;
        const NodeInfo &na = nodes_[a], &nb = nodes_[b];
        NodeInfo& nr = nodes_[r];
        nr.var_mask = na.var_mask | nb.var_mask;
        nr.level = std::max(na.level, nb.level);
        nr.pass_dep = na.pass_dep || nb.pass_dep;
        nr.slice_mask = na.slice_mask | nb.slice_mask;
        nr.cfg_dep = na.cfg_dep || nb.cfg_dep;
        StepInfo st;
        st.plan_index = step_origin_.empty() ? s : step_origin_[s];
        st.a = a;
        st.b = b;
        st.r = r;
        st.level = nr.level;
        st.phase = nr.level < 2 ? nr.level : (nr.pass_dep ? 2 : 3);
        nodes_[a].consumer = s;
        nodes_[b].consumer = s;
        steps_.push_back(st);
        // result layout is decided in build_steps (needs operand roles)
        nr.labels.clear();
    }
    root_ = plan.n_steps ? plan.steps[3 * (plan.n_steps - 1) + 2] : 0;
    if (plan.n_steps == 0 && net.n_leaves != 1)
        throw Failure{RCSG_ERR_CONFIG, "plan has no steps but the network has several tensors"};
    for (int i = 0; i < n_nodes; ++i)
        if (i != root_ && made[i] && !used[i])
            throw Failure{RCSG_ERR_CONFIG, "plan leaves node " + std::to_string(i) + " unconsumed"};
}

void Program::build_steps() {
    // Consumer-driven layouts.  Every operand is consumed as [kept labels |
    // contracted labels] (K-major GEMM operands).  Steps are planned from the
    // root backwards: each step fixes the layout of its two operands, and the
    // producer of an operand (a GEMM epilogue or the leaf projection) writes its
    // result directly in that layout through a bit-scatter store map, so no
    // intermediate tensor is ever permuted.  Key choices:
    //   * M side: the group-variant operand (variants fold into M), else the
    //     operand with more kept labels;
    //   * kept-label orders end with the run of output bits the consumer needs
    //     fastest, so the epilogue's stores stay coalesced;
    //   * the contraction order puts last the shared labels that sit on the same
    //     side of both producers (their fastest output bits).
    const int n_nodes = static_cast<int>(nodes_.size());
    std::vector<std::vector<int>> lset(n_nodes);
    for (int i = 0; i < n_leaves_; ++i) {
        lset[i] = nodes_[i].labels;
        std::sort(lset[i].begin(), lset[i].end());
    }
    std::vector<int> producer(n_nodes, -1);
    std::vector<std::vector<int>> keep_m(steps_.size()), keep_n(steps_.size()), shared(steps_.size());
    for (size_t s = 0; s < steps_.size(); ++s) {
        StepInfo& st = steps_[s];
        std::vector<int> sh, kx, ky;
        std::set_intersection(lset[st.a].begin(), lset[st.a].end(), lset[st.b].begin(), lset[st.b].end(),
                              std::back_inserter(sh));
        std::set_difference(lset[st.a].begin(), lset[st.a].end(), sh.begin(), sh.end(), std::back_inserter(kx));
        std::set_difference(lset[st.b].begin(), lset[st.b].end(), sh.begin(), sh.end(), std::back_inserter(ky));
        const bool vx = nodes_[st.a].level == 2, vy = nodes_[st.b].level == 2;
        bool swap = false;
        if (vy && !vx) swap = true;
        else if (vx == vy && ky.size() > kx.size()) swap = true;
        if (swap) {
            std::swap(st.a, st.b);
            std::swap(kx, ky);
        }
        st.mode = nodes_[st.a].level == 2 ? (nodes_[st.b].level == 2 ? 2 : 1) : 0;
        keep_m[s] = kx;
        keep_n[s] = ky;
        shared[s] = sh;
        std::set_symmetric_difference(lset[st.a].begin(), lset[st.a].end(), lset[st.b].begin(), lset[st.b].end(),
                                      std::back_inserter(lset[st.r]));
        producer[st.r] = static_cast<int>(s);
    }
    // side of label l in the output of node `id`'s producer: 0 M, 1 N, 2 leaf
    auto side = [&](int id, int l) {
        const int p = producer[id];
        if (p < 0) return 2;
        return std::binary_search(keep_m[p].begin(), keep_m[p].end(), l) ? 0 : 1;
    };
    std::vector<std::vector<int>> layout(n_nodes);  // required (or chosen) layout of every node
    std::vector<std::vector<int>> ord_m(steps_.size()), ord_n(steps_.size());
    for (int s = static_cast<int>(steps_.size()) - 1; s >= 0; --s) {
        StepInfo& st = steps_[s];
        std::vector<int>& L = layout[st.r];
        if (L.empty()) {  // the root: any layout (finalize reads it through a map)
            L = keep_m[s];
            L.insert(L.end(), keep_n[s].begin(), keep_n[s].end());
        }
        // kept-label orders: the output's fastest run (one side) goes last on its side
        auto in = [](const std::vector<int>& v, int l) { return std::binary_search(v.begin(), v.end(), l); };
        std::vector<int> om, on;
        for (int l : L) (in(keep_m[s], l) ? om : on).push_back(l);
        if (!L.empty()) {
            const bool last_m = in(keep_m[s], L.back());
            std::vector<int> tail;
            for (auto it = L.rbegin(); it != L.rend() && in(last_m ? keep_m[s] : keep_n[s], *it) == true; ++it)
                tail.insert(tail.begin(), *it);
            std::vector<int>& side_ord = last_m ? om : on;
            std::vector<int> head;
            for (int l : side_ord)
                if (std::find(tail.begin(), tail.end(), l) == tail.end()) head.push_back(l);
            head.insert(head.end(), tail.begin(), tail.end());
            side_ord = head;
        }
        ord_m[s] = om;
        ord_n[s] = on;
        // contraction order: the largest group of shared labels lying on the same
        // side of both producers goes last (fastest), canonical inside groups
        std::map<int, std::vector<int>> groups;
        for (int l : shared[s]) groups[side(st.a, l) * 3 + side(st.b, l)].push_back(l);
        // score: run length (capped at the 32-element coalescing width), then
        // prefer the producers' column side (all epilogues store columns
        // contiguously; row-fast stores need the row-mode kernels)
        int best_key = -1;
        double best_score = -1;
        for (auto& [k, v] : groups) {
            const int sa = k / 3, sb = k % 3;
            const double score = std::min<size_t>(v.size(), 5) * 10.0 + (sa != 0) + (sb != 0) + 0.01 * v.size();
            if (score > best_score) {
                best_score = score;
                best_key = k;
            }
        }
        std::vector<int> sigma;
        for (auto& [k, v] : groups)
            if (k != best_key) sigma.insert(sigma.end(), v.begin(), v.end());
        if (best_key >= 0) sigma.insert(sigma.end(), groups[best_key].begin(), groups[best_key].end());
        layout[st.a] = om;
        layout[st.a].insert(layout[st.a].end(), sigma.begin(), sigma.end());
        layout[st.b] = on;
        layout[st.b].insert(layout[st.b].end(), sigma.begin(), sigma.end());
    }
    // leaves take their required layouts (the leaf projection writes them)
    for (int i = 0; i < n_leaves_; ++i)
        if (!layout[i].empty()) nodes_[i].labels = layout[i];
    // forward: operand layouts, GEMM shapes, output scatter maps.  RCSG_FORCE_PERMUTE=1
    // (tests only) makes every step write its natural [rows | cols] order so the
    // consumers run the bit-permutation kernel instead of the scatter epilogue.
    const bool force_permute = getenv("RCSG_FORCE_PERMUTE") && atoi(getenv("RCSG_FORCE_PERMUTE")) != 0;
    for (size_t s = 0; s < steps_.size(); ++s) {
        StepInfo& st = steps_[s];
        NodeInfo& A = nodes_[st.a];
        NodeInfo& B = nodes_[st.b];
        std::vector<int> ta = ord_m[s], tb = ord_n[s];
        const std::vector<int> sigma(layout[st.a].end() - shared[s].size(), layout[st.a].end());
        ta.insert(ta.end(), sigma.begin(), sigma.end());
        tb.insert(tb.end(), sigma.begin(), sigma.end());
        std::vector<int> bits;
        st.perm_a = ta != A.labels;  // only if a producer could not comply (should not happen)
        if (st.perm_a) {
            permute_bits(A.labels, ta, bits);
            st.pa = make_permute(static_cast<int>(ta.size()), bits.data());
        }
        st.perm_b = tb != B.labels;
        if (st.perm_b) {
            permute_bits(B.labels, tb, bits);
            st.pb = make_permute(static_cast<int>(tb.size()), bits.data());
        }
        st.m = int64_t{1} << ord_m[s].size();
        st.n = int64_t{1} << ord_n[s].size();
        st.k = int64_t{1} << shared[s].size();
        st.flops_per_variant = 8ull * st.m * st.n * st.k;
        plan_flops_ += st.flops_per_variant;
        NodeInfo& R = nodes_[st.r];
        R.labels = layout[st.r];
        if (force_permute) {  // test knob: results in GEMM order, consumers transpose (permute.cu)
            R.labels = ord_m[s];
            R.labels.insert(R.labels.end(), ord_n[s].begin(), ord_n[s].end());
        }
        if (R.labels.size() > static_cast<size_t>(kMaxRank))
            throw Failure{RCSG_ERR_CAPACITY, "intermediate rank exceeds the executor limit"};
        R.payload = int64_t{1} << R.labels.size();
        // scatter map: bit j of the row index (LSB = last label of ord_m) -> output bit
        OutMap& om = st.om;
        om.m_bits = static_cast<int32_t>(ord_m[s].size());
        om.n_bits = static_cast<int32_t>(ord_n[s].size());
        const int rr = static_cast<int>(R.labels.size());
        bool ident = true;
        for (int j = 0; j < om.m_bits; ++j) {
            const int l = ord_m[s][om.m_bits - 1 - j];
            om.m_pos[j] = static_cast<int8_t>(rr - 1 - pos_in(R.labels, l));
            ident &= om.m_pos[j] == j + om.n_bits;
        }
        for (int j = 0; j < om.n_bits; ++j) {
            const int l = ord_n[s][om.n_bits - 1 - j];
            om.n_pos[j] = static_cast<int8_t>(rr - 1 - pos_in(R.labels, l));
            ident &= om.n_pos[j] == j;
        }
        om.scatter = ident ? 0 : 1;
        if (getenv("RCSG_DUMP_STEPS") && (A.labels.size() >= 16 || B.labels.size() >= 16 || R.labels.size() >= 20))
            fprintf(stderr, "step %d mode %d m=2^%d n=2^%d k=2^%zu perm_a %d perm_b %d scatter %d low-bit m_pos0=%d n_pos0=%d\n",
                    st.plan_index, st.mode, om.m_bits, om.n_bits, shared[s].size(), st.perm_a, st.perm_b,
                    om.scatter, om.m_bits ? om.m_pos[0] : -1, om.n_bits ? om.n_pos[0] : -1);
        if (getenv("RCSG_DUMP_STEPS") && R.labels.size() >= 20) {
            fprintf(stderr, "   m_pos:");
            for (int j = 0; j < om.m_bits; ++j) fprintf(stderr, " %d", om.m_pos[j]);
            fprintf(stderr, "\n   n_pos:");
            for (int j = 0; j < om.n_bits; ++j) fprintf(stderr, " %d", om.n_pos[j]);
            fprintf(stderr, "\n");
        }
    }
    // canonical output order of the root: bit j <-> j-th smallest open qubit
    // among the root's labels (contraction_engine.cpp:193-207)
    const NodeInfo& root = nodes_[root_];
    out_rank_ = static_cast<int>(root.labels.size());
    std::vector<std::pair<int, int>> q_pos;  // (qubit, layout position)
    for (int p = 0; p < out_rank_; ++p) {
        const int q = canon_qubit_[root.labels[p]];
        if (q < 0)
            throw Failure{RCSG_ERR_CONFIG, "free label " + std::to_string(root.labels[p]) +
                                               " is not an open output; assignment incomplete"};
        q_pos.push_back({q, p});
    }
    std::sort(q_pos.begin(), q_pos.end());
    root_canon_src_.assign(out_rank_, 0);
    for (int j = 0; j < out_rank_; ++j) root_canon_src_[j] = out_rank_ - 1 - q_pos[j].second;
}

// Arena layout by first-fit simulation of one run's leveled schedule.
int64_t Program::plan_arena(int64_t cap, bool assign) {
    FirstFit ff;
    auto var_cap = [&](const NodeInfo& nd) -> int64_t {
        if (nd.level < 2) return 1;
        const int bits = __builtin_popcountll(nd.var_mask);
        return bits >= 62 ? cap : std::min<int64_t>(cap, int64_t{1} << bits);
    };
    auto place = [&](int id) {
        NodeInfo& nd = nodes_[id];
        nd.max_var = var_cap(nd);
        nd.plane = align_up(nd.max_var * nd.payload);
        nd.off = ff.alloc(2 * nd.plane);
    };
    // leaves: persistent
    for (int i = 0; i < n_leaves_; ++i) place(i);
    // phases in execution order: constant (0), group-only (3; cached when the
    // groups fit one chunk), per pass (1), per pass and group (2).  Results
    // consumed by a later phase persist; per-pass results read by phase 2
    // persist until the pass ends.
    auto phase_of = [&](const NodeInfo& nd) {
        if (nd.tab && !nd.is_leaf) return 4;  // slice-table steps (their own phase, see below)
        return nd.level < 2 ? nd.level : (nd.pass_dep ? 2 : 3);
    };
    // the slice-table steps (phase 4) run before phase 1 in the simulation: their
    // intermediates are free again afterwards, and the boundary nodes (gathered
    // at pass start) stay allocated until their per-pass consumers run
    // one chunk: group-only results (phase 3) are computed once, before the
    // passes; several chunks: each pass recomputes them per chunk after phase 1,
    // so the simulation must follow that order (phase-3 intermediates may then
    // not reuse memory of still-live per-pass results)
    const bool multi_chunk = cap < plan_codes_;
    std::vector<int> persist_until_pass_end;
    const std::vector<int> order = multi_chunk ? std::vector<int>{0, 4, 1, 3, 2} : std::vector<int>{0, 3, 4, 1, 2};
    for (int ph : order) {
        for (StepInfo& st : steps_) {
            if ((st.tab ? 4 : st.phase) != ph) continue;
            const NodeInfo &A = nodes_[st.a], &B = nodes_[st.b];
            if (st.perm_a) {
                st.sa_plane = align_up(var_cap(A) * A.payload);
                st.sa_off = ff.alloc(2 * st.sa_plane);
            }
            if (st.perm_b) {
                st.sb_plane = align_up(var_cap(B) * B.payload);
                st.sb_off = ff.alloc(2 * st.sb_plane);
            }
            place(st.r);
            if (st.perm_a) ff.release(st.sa_off, 2 * st.sa_plane);
            if (st.perm_b) ff.release(st.sb_off, 2 * st.sb_plane);
            for (int op : {st.a, st.b}) {
                NodeInfo& o = nodes_[op];
                if (o.is_leaf) continue;
                if (phase_of(o) == ph) ff.release(o.off, 2 * o.plane);
                else if (phase_of(o) == 4 && ph == 2) persist_until_pass_end.push_back(op);  // boundary node
                else if (phase_of(o) == 4) ff.release(o.off, 2 * o.plane);  // boundary node, consumed in phase 1
                else if (phase_of(o) == 1 && ph == 2) persist_until_pass_end.push_back(op);
                // constant and group-only operands of later phases persist for the run
            }
        }
        if (ph == 2) {
            // the root is read by the finalize of every chunk
            if (phase_of(nodes_[root_]) == 2 && !nodes_[root_].is_leaf)
                ff.release(nodes_[root_].off, 2 * nodes_[root_].plane);
            for (int id : persist_until_pass_end) ff.release(nodes_[id].off, 2 * nodes_[id].plane);
        }
    }
    (void)assign;
    return ff.peak;
}

void Program::free_chunks() {
    for (ChunkData& c : chunks_) {
        cudaFree(c.d_codes);
        cudaFree(c.d_idx);
        cudaFree(c.d_fin);
        cudaFree(c.d_leaf_jobs);
    }
    chunks_.clear();
}

void Program::prepare_chunks(const std::vector<uint64_t>& groups, int64_t cap) {
    free_chunks();
    // distinct group codes, ascending; duplicates share every variant
    std::vector<uint64_t> uniq = groups;
    std::sort(uniq.begin(), uniq.end());
    uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
    std::map<uint64_t, std::vector<int32_t>> members;
    for (size_t g = 0; g < groups.size(); ++g) members[groups[g]].push_back(static_cast<int32_t>(g));
    const int64_t n_nodes = static_cast<int64_t>(nodes_.size());
    for (size_t u0 = 0; u0 < uniq.size(); u0 += static_cast<size_t>(cap)) {
        const size_t u1 = std::min(uniq.size(), u0 + static_cast<size_t>(cap));
        ChunkData ch;
        ch.codes_off.assign(n_nodes, -1);
        ch.nvar.assign(n_nodes, 1);
        std::vector<std::vector<uint64_t>> node_codes(n_nodes);
        for (int64_t i = 0; i < n_nodes; ++i) {
            const NodeInfo& nd = nodes_[i];
            if (nd.level != 2) continue;
            std::vector<uint64_t>& c = node_codes[i];
            for (size_t u = u0; u < u1; ++u) c.push_back(uniq[u] & nd.var_mask);
            std::sort(c.begin(), c.end());
            c.erase(std::unique(c.begin(), c.end()), c.end());
            ch.codes_off[i] = static_cast<int64_t>(ch.codes.size());
            ch.nvar[i] = static_cast<int64_t>(c.size());
            ch.codes.insert(ch.codes.end(), c.begin(), c.end());
        }
        auto find_code = [&](int node, uint64_t code) -> int32_t {
            const auto& c = node_codes[node];
            return static_cast<int32_t>(std::lower_bound(c.begin(), c.end(), code) - c.begin());
        };
        ch.ia_off.assign(steps_.size(), -1);
        ch.ib_off.assign(steps_.size(), -1);
        ch.perm_off.assign(steps_.size(), -1);
        for (size_t s = 0; s < steps_.size(); ++s) {
            const StepInfo& st = steps_[s];
            if (st.mode != 2) continue;
            ch.ia_off[s] = static_cast<int64_t>(ch.idx.size());
            for (uint64_t c : node_codes[st.r]) ch.idx.push_back(find_code(st.a, c & nodes_[st.a].var_mask));
            ch.ib_off[s] = static_cast<int64_t>(ch.idx.size());
            for (uint64_t c : node_codes[st.r]) ch.idx.push_back(find_code(st.b, c & nodes_[st.b].var_mask));
            const int64_t va = ch.nvar[st.a], vb = ch.nvar[st.b], vr = ch.nvar[st.r];
            if (vr < 2 || va * vb == vr) continue;  // full products: product_order
            {
                // an operand with fewer variants than the result, at least 4x larger per
                // variant than the other: order the results by its variant so that the
                // GEMM's tiles in flight share its panels (RCSG_NO_VPERM: off)
                const double sa = static_cast<double>(st.m) * st.k, sb = static_cast<double>(st.n) * st.k;
                const bool by_a = va < vr && sa >= 4 * sb, by_b = vb < vr && sb >= 4 * sa;
                if ((by_a || by_b) && !getenv("RCSG_NO_VPERM")) {
                    const int64_t off_s = by_a ? ch.ia_off[s] : ch.ib_off[s], off_o = by_a ? ch.ib_off[s] : ch.ia_off[s];
                    std::vector<int32_t> order(static_cast<size_t>(vr));
                    std::iota(order.begin(), order.end(), 0);
                    std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) {
                        const int32_t sx = ch.idx[off_s + x], sy = ch.idx[off_s + y];
                        return sx != sy ? sx < sy : ch.idx[off_o + x] < ch.idx[off_o + y];
                    });
                    ch.perm_off[s] = static_cast<int64_t>(ch.idx.size());
                    ch.idx.insert(ch.idx.end(), order.begin(), order.end());
                    if (getenv("RCSG_DEBUG_VPERM"))
                        fprintf(stderr, "[rcsg] vperm step %d by %c va %lld vb %lld vr %lld\n", st.plan_index,
                                by_a ? 'A' : 'B', (long long)va, (long long)vb, (long long)vr);
                }
            }
        }
        const int64_t G = static_cast<int64_t>(n_ext_groups_);
        std::vector<std::array<int32_t, 3>> ent;  // (group, lo, root variant)
        for (size_t u = u0; u < u1; ++u)
            for (int32_t c : members[uniq[u]])
                ent.push_back({static_cast<int32_t>(c % G), static_cast<int32_t>(c / G),
                               nodes_[root_].level == 2 ? find_code(root_, uniq[u] & nodes_[root_].var_mask) : 0});
        std::sort(ent.begin(), ent.end());
        for (size_t e = 0; e < ent.size(); ++e) {
            if (e == 0 || ent[e][0] != ent[e - 1][0]) {
                ch.fin_g.push_back(ent[e][0]);
                ch.fin_off.push_back(static_cast<int32_t>(e));
            }
            ch.ent_lo.push_back(ent[e][1]);
            ch.ent_vid.push_back(ent[e][2]);
        }
        ch.fin_off.push_back(static_cast<int32_t>(ent.size()));
        // level-2 leaf jobs of this chunk: group-only leaves, then pass-dependent ones
        std::vector<LeafJob> jobs;
        std::vector<int> leaf_order;
        for (int want_pass = 0; want_pass < 2; ++want_pass)
            for (int i = 0; i < n_leaves_; ++i)
                if (nodes_[i].level == 2 && nodes_[i].pass_dep == (want_pass == 1)) leaf_order.push_back(i);
        for (int i : leaf_order) {
            const NodeInfo& nd = nodes_[i];
            if (!nd.pass_dep) ++ch.n_leaf_jobs3;
            LeafJob j{};
            j.out_off = nd.off;
            j.out_plane = nd.plane;
            j.data_off = nd.data_off;
            j.rank = nd.rank0;
            j.out_rank = static_cast<int32_t>(nd.labels.size());
            j.n_var = static_cast<int32_t>(ch.nvar[i]);
            j.codes_off = static_cast<int32_t>(ch.codes_off[i]);
            for (int p = 0; p < nd.rank0; ++p) {
                const LabelRole& rl = roles_[nd.labels0[p]];
                j.kind[p] = rl.role;
                j.arg[p] = static_cast<int16_t>(rl.role == kVar ? rl.var_bit : nd.labels0[p]);
                j.obit[p] = rl.role == kFree ? static_cast<int8_t>(nd.labels.size() - 1 - pos_in(nd.labels, nd.labels0[p])) : 0;
            }
            jobs.push_back(j);
        }
        ch.n_leaf_jobs = static_cast<int>(jobs.size());
        CUDA_OK(cudaMalloc(&ch.d_codes, std::max<size_t>(ch.codes.size(), 1) * sizeof(uint64_t)));
        CUDA_OK(cudaMemcpy(ch.d_codes, ch.codes.data(), ch.codes.size() * sizeof(uint64_t), cudaMemcpyHostToDevice));
        CUDA_OK(cudaMalloc(&ch.d_idx, std::max<size_t>(ch.idx.size(), 1) * sizeof(int32_t)));
        CUDA_OK(cudaMemcpy(ch.d_idx, ch.idx.data(), ch.idx.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
        {
            std::vector<int32_t> fin = ch.fin_g;
            fin.insert(fin.end(), ch.fin_off.begin(), ch.fin_off.end());
            fin.insert(fin.end(), ch.ent_vid.begin(), ch.ent_vid.end());
            fin.insert(fin.end(), ch.ent_lo.begin(), ch.ent_lo.end());
            CUDA_OK(cudaMalloc(&ch.d_fin, fin.size() * sizeof(int32_t)));
            CUDA_OK(cudaMemcpy(ch.d_fin, fin.data(), fin.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
        }
        CUDA_OK(cudaMalloc(&ch.d_leaf_jobs, std::max<size_t>(jobs.size(), 1) * sizeof(LeafJob)));
        CUDA_OK(cudaMemcpy(ch.d_leaf_jobs, jobs.data(), jobs.size() * sizeof(LeafJob), cudaMemcpyHostToDevice));
        chunks_.push_back(std::move(ch));
    }
}

void* Program::buf(int64_t off) const {
    return static_cast<char*>(arena_) + off * elem_bytes_;
}

// GEMM arguments of a step on its (unpermuted) operand buffers
GemmArgs Program::step_args(const StepInfo& st, const ChunkData* ch) const {
    const NodeInfo &A = nodes_[st.a], &B = nodes_[st.b], &Rn = nodes_[st.r];
    const int64_t va = (A.level == 2 && ch) ? ch->nvar[st.a] : 1;
    const int64_t vr = (Rn.level == 2 && ch) ? ch->nvar[st.r] : 1;
    GemmArgs g{};
    g.a = buf(A.off);
    g.a_plane = A.plane;
    g.b = buf(B.off);
    g.b_plane = B.plane;
    g.c = buf(Rn.off);
    g.c_plane = Rn.plane;
    g.k = st.k;
    g.n = st.n;
    g.step = st.plan_index;
    g.fault = d_fault_;
    g.om = st.om;
    g.scale_exp = node_exp_[st.a] + node_exp_[st.b] - node_exp_[st.r];
    static const bool chop = getenv("RCSG_TF32_CHOP") != nullptr;  // probes: the MMA's own truncation
    g.round_tf32 = precision_ == RCSG_PREC_TF32 && !chop;
    g.split_tf32 = precision_ == RCSG_PREC_3XTF32;
    const int64_t vb = (B.level == 2 && ch) ? ch->nvar[st.b] : 1;
    const int prod = st.mode == 2 ? product_order(A.var_mask, B.var_mask, va, vb, vr) : 0;
    if (prod) {
        // every (A variant, B variant) pair is a result variant and one operand's
        // code bits lie above the other's: the variants fold into M and N of one
        // GEMM, result variant = b * va + a (B high) or a * vb + b (A high)
        const int64_t mn = st.m * st.n;
        g.m = st.m * va;
        g.n = st.n * vb;
        g.batch = 1;
        if (!g.om.scatter) {  // identity layout as an explicit map
            g.om.scatter = 1;
            for (int j = 0; j < g.om.n_bits; ++j) g.om.n_pos[j] = static_cast<int8_t>(j);
            for (int j = 0; j < g.om.m_bits; ++j) g.om.m_pos[j] = static_cast<int8_t>(g.om.n_bits + j);
        }
        g.om.m_vstride = prod == 2 ? mn : vb * mn;
        g.om.n_vstride = prod == 2 ? va * mn : mn;
    } else if (st.mode == 2) {
        g.m = st.m;
        g.batch = vr;
        g.a_batch = st.m * st.k;
        g.b_batch = st.n * st.k;
        g.c_batch = st.m * st.n;
        g.ia = ch->d_idx + ch->ia_off[&st - steps_.data()];
        g.ib = ch->d_idx + ch->ib_off[&st - steps_.data()];
        if (ch->perm_off[&st - steps_.data()] >= 0) g.vperm = ch->d_idx + ch->perm_off[&st - steps_.data()];
    } else {
        g.m = st.m * va;  // mode 1: the variants fold into M
        g.batch = 1;
    }
    return g;
}

// 0: not a full product; 1: A's code bits above B's; 2: B's above A's
int Program::product_order(uint64_t ma, uint64_t mb, int64_t va, int64_t vb, int64_t vr) {
    if (!ma || !mb || vr != va * vb) return 0;
    const int hi_a = 63 - __builtin_clzll(ma), lo_a = __builtin_ctzll(ma);
    const int hi_b = 63 - __builtin_clzll(mb), lo_b = __builtin_ctzll(mb);
    if (lo_a > hi_b) return 1;
    if (lo_b > hi_a) return 2;
    return 0;
}

template <typename R>
void Program::exec_step_t(const StepInfo& st, const ChunkData* ch) {
    const NodeInfo &A = nodes_[st.a], &B = nodes_[st.b], &Rn = nodes_[st.r];
    const int64_t va = (A.level == 2 && ch) ? ch->nvar[st.a] : 1;
    const int64_t vb = (B.level == 2 && ch) ? ch->nvar[st.b] : 1;
    const int64_t vr = (Rn.level == 2 && ch) ? ch->nvar[st.r] : 1;
    const R* a_ptr = static_cast<const R*>(buf(A.off));
    int64_t a_plane = A.plane;
    if (st.perm_a) {
        R* dst = static_cast<R*>(buf(st.sa_off));
        const int mk = mark_begin();
        launch_permute<R>(a_ptr, A.plane, dst, st.sa_plane, va, st.pa, ls_);
        mark_end(mk, kCatPermute, 4ull * sizeof(R) * va * A.payload, st.plan_index, va, A.payload, 0, 0);
        ++launches_;
        a_ptr = dst;
        a_plane = st.sa_plane;
    }
    const R* b_ptr = static_cast<const R*>(buf(B.off));
    int64_t b_plane = B.plane;
    if (st.perm_b) {
        R* dst = static_cast<R*>(buf(st.sb_off));
        const int mk = mark_begin();
        launch_permute<R>(b_ptr, B.plane, dst, st.sb_plane, vb, st.pb, ls_);
        mark_end(mk, kCatPermute, 4ull * sizeof(R) * vb * B.payload, st.plan_index, vb, B.payload, 0, 0);
        ++launches_;
        b_ptr = dst;
        b_plane = st.sb_plane;
    }
    GemmArgs g = step_args(st, ch);
    g.a = a_ptr;
    g.a_plane = a_plane;
    g.b = b_ptr;
    g.b_plane = b_plane;
    const uint64_t flops = st.flops_per_variant * static_cast<uint64_t>(vr);
    exec_flops_ += flops;
    if (profile_ && getenv("RCSG_DUMP_VARS") && flops > (1ull << 32))
        fprintf(stderr, "[rcsg] step %d mode %d va %lld vb %lld vr %lld m %lld n %lld k %lld\n", st.plan_index, st.mode,
                (long long)va, (long long)vb, (long long)vr, (long long)st.m, (long long)st.n, (long long)st.k);
    if (profile_ && getenv("RCSG_DUMP_VARS") && flops > (1ull << 32) && st.mode == 2 && ch) {
        const size_t si = static_cast<size_t>(&st - steps_.data());
        fprintf(stderr, "[rcsg]   ia:");
        for (int64_t v = 0; v < std::min<int64_t>(vr, 20); ++v) fprintf(stderr, " %d", ch->idx[ch->ia_off[si] + v]);
        fprintf(stderr, "\n[rcsg]   ib:");
        for (int64_t v = 0; v < std::min<int64_t>(vr, 20); ++v) fprintf(stderr, " %d", ch->idx[ch->ib_off[si] + v]);
        fprintf(stderr, "\n");
    }
    const int mk = mark_begin();
    if (mk >= 0) {  // algorithmic bytes: every operand variant read once, the result written once
        const int64_t eb = 2 * elem_bytes_;
        marks_[mk].bytes = static_cast<uint64_t>(eb * (va * st.m * st.k + vb * st.n * st.k + vr * st.m * st.n));
    }
    const bool tc_ok = !std::is_same_v<R, double> &&
                       (precision_ == RCSG_PREC_TF32 || precision_ == RCSG_PREC_3XTF32 ||
                        precision_ >= RCSG_PREC_BF16) &&
                       gemm_tc_supported(g);
    // K <= 16 goes to the register-blocked outer-product kernel, except large
    // K = 5..16 products, which are CUDA-core FMA-bound there and memory-bound
    // on the tensor cores (narrow-K tiles zero-fill K up to 16)
    static const int64_t smallk_max_n = getenv("RCSG_SMALLK_MAXN") ? atoll(getenv("RCSG_SMALLK_MAXN")) : 0;
    const bool big_k16 = g.k > 4 && static_cast<double>(g.m) * g.n * std::max<int64_t>(g.batch, 1) >= 4194304.0 &&
                         !(std::min(g.m, g.n) <= smallk_max_n);
    if (gemm_smallk_supported(g) && !(tc_ok && big_k16)) {
        launch_gemm_smallk<R>(g, ls_);
        mark_end(mk, kCatGemmSimt, flops, st.plan_index, g.m, g.n, g.k, g.batch);
        ++launches_;
        return;
    }
    if (gemv_supported(g)) {
        launch_gemv<R>(g, ls_);
        mark_end(mk, kCatGemv, flops, st.plan_index, g.m, g.n, g.k, g.batch);
        ++launches_;
        return;
    }
    if constexpr (!std::is_same_v<R, double>) {
        // tf32, fp16, bf16 and 3xtf32 (split fp32 operands, gemm_tc.cu launch_split) on tcgen05
        if (tc_ok) {
            launch_gemm_tc(g, precision_ == RCSG_PREC_BF16 ? 1 : (precision_ == RCSG_PREC_F16 ? 2 : 0), ls_);
            mark_end(mk, kCatGemmTc, flops, st.plan_index, g.m, g.n, g.k, g.batch);
            ++launches_;
            return;
        }
    }
    launch_gemm_simt<R>(g, ls_);
    mark_end(mk, kCatGemmSimt, flops, st.plan_index, g.m, g.n, g.k, g.batch);
    ++launches_;
}

int Program::mark_begin() {
    if (!profile_) return -1;
    const size_t i = marks_.size();
    if (ev_pool_.size() < 2 * (i + 1)) {
        cudaEvent_t a, b;
        CUDA_OK(cudaEventCreate(&a));
        CUDA_OK(cudaEventCreate(&b));
        ev_pool_.push_back(a);
        ev_pool_.push_back(b);
    }
    marks_.push_back({-1, 0, -1, 0, 0, 0, 0});
    CUDA_OK(cudaEventRecord(ev_pool_[2 * i], ls_));
    return static_cast<int>(i);
}

void Program::mark_end(int idx, int cat, uint64_t work, int step, int64_t m, int64_t n, int64_t k,
                       int64_t batch) {
    if (idx < 0) return;
    const uint64_t bytes = marks_[idx].bytes;
    marks_[idx] = {cat, work, step, m, n, k, batch, bytes};
    CUDA_OK(cudaEventRecord(ev_pool_[2 * idx + 1], ls_));
}

void Program::collect_marks(rcsg_stats* stats) {
    // RCSG_PROFILE_STEPS=N prints the N most expensive launches (stderr)
    const char* env = getenv("RCSG_PROFILE_STEPS");
    std::vector<std::pair<float, size_t>> order;
    const int64_t prev_top = stats ? stats->top_step : -1;
    for (size_t i = 0; i < marks_.size(); ++i) {
        float ms = 0;
        CUDA_OK(cudaEventElapsedTime(&ms, ev_pool_[2 * i], ev_pool_[2 * i + 1]));
        order.push_back({ms, i});
        if (!stats) continue;
        const Mark& m = marks_[i];
        if (m.cat == kCatGemmSimt || m.cat == kCatGemmTc || m.cat == kCatGemv) stats->gemm_ms += ms;
        if (m.cat == kCatGemmTc) {
            stats->gemm_tc_ms += ms;
            stats->gemm_tc_flops += m.work;
            stats->gemm_tc_launches += 1;
        }
        if (m.cat == kCatPermute) {
            stats->permute_ms += ms;
            stats->permute_bytes += m.work;
        }
        if (ms > stats->top_ms) {
            stats->top_ms = ms;
            stats->top_flops = m.cat == kCatPermute ? 0 : m.work;
            stats->top_bytes = m.cat == kCatPermute ? m.work : m.bytes;
            stats->top_step = m.step;
            stats->top_class = m.cat;
        }
    }
    if (stats) {  // every launch of the dominant plan step: its average launch time
        if (stats->top_step != prev_top) {
            stats->top_ms_sum = 0;
            stats->top_launches = 0;
        }
        for (const auto& [ms, i] : order)
            if (marks_[i].step == stats->top_step && marks_[i].cat == stats->top_class) {
                stats->top_ms_sum += ms;
                stats->top_launches += 1;
            }
    }
    if (getenv("RCSG_PROFILE_ORDER")) {  // every launch in issue order (joins an ncu launch list)
        static const char* cats[] = {"gemm_simt", "gemm_tc", "permute", "gemv"};
        for (size_t i = 0; i < marks_.size(); ++i) {
            const Mark& m = marks_[i];
            fprintf(stderr, "[rcsg-order] %zu %s %d %lld %lld %lld %lld %.6e %.6e %.6f\n", i,
                    m.cat >= 0 ? cats[m.cat] : "?", m.step, (long long)m.m, (long long)m.n, (long long)m.k,
                    (long long)m.batch, (double)m.work, (double)m.bytes, order[i].first);
        }
    }
    if (env) {
        std::sort(order.rbegin(), order.rend());
        static const char* names[] = {"gemm_simt", "gemm_tc", "permute", "gemv"};
        const size_t top = std::min<size_t>(order.size(), static_cast<size_t>(atoi(env)));
        for (size_t j = 0; j < top; ++j) {
            const Mark& m = marks_[order[j].second];
            const double sec = order[j].first * 1e-3;
            fprintf(stderr,
                    "[rcsg] %8.3f ms %-9s step %4d m=%lld n=%lld k=%lld batch=%lld work=%.3e bytes=%.3e "
                    "%.1f TF/s %.1f GB/s\n",
                    order[j].first, m.cat >= 0 ? names[m.cat] : "?", m.step, (long long)m.m, (long long)m.n,
                    (long long)m.k, (long long)m.batch, (double)m.work, (double)m.bytes,
                    sec > 0 ? (double)m.work / sec * 1e-12 : 0.0, sec > 0 ? (double)m.bytes / sec * 1e-9 : 0.0);
        }
    }
    marks_.clear();
}

void Program::exec_step(const StepInfo& st, const ChunkData* ch) {
    RCSG_DISPATCH(precision_, exec_step_t<S>(st, ch));
    if (record_max_) {  // calibration: max |value| of the step's output
        const NodeInfo& R = nodes_[st.r];
        const int64_t vr = (R.level == 2 && ch) ? ch->nvar[st.r] : 1;
        launch_maxabs(static_cast<const float*>(buf(R.off)), R.plane, vr * R.payload, d_max_ + st.r, ls_);
    }
}

void Program::exec_phase(int phase, const ChunkData* ch) {
    // leaves of this phase
    if (phase < 2) {
        if (!static_jobs_[phase].empty()) {
            RCSG_DISPATCH(precision_, launch_leaf_project<S>(d_static_jobs_[phase],
                                                            static_cast<int>(static_jobs_[phase].size()),
                                                            d_leaf_data_, nullptr, d_pass_src_, d_state_,
                                                            static_cast<S*>(arena_), ls_, round_leaves()));
            ++launches_;
        }
    } else {
        const int j0 = phase == 3 ? 0 : ch->n_leaf_jobs3;
        const int j1 = phase == 3 ? ch->n_leaf_jobs3 : ch->n_leaf_jobs;
        if (j1 > j0) {
            RCSG_DISPATCH(precision_, launch_leaf_project<S>(ch->d_leaf_jobs + j0, j1 - j0, d_leaf_data_, ch->d_codes,
                                                            d_pass_src_, d_state_, static_cast<S*>(arena_), ls_, round_leaves()));
            ++launches_;
        }
    }
    if (phase == 1 && !tab_jobs_.empty()) {  // this pass's entries of the slice tables
        launch_table_io(d_tab_jobs_, static_cast<int>(tab_jobs_.size()), d_state_, arena_, elem_bytes_, 0, ls_);
        ++launches_;
    }
    for (const StepInfo& st : steps_)
        if (st.phase == phase && !st.tab) exec_step(st, ch);
}

void Program::run(const std::vector<uint64_t>& groups, const std::vector<uint64_t>& configs,
                  uint64_t slice_begin, uint64_t slice_end, double* d_acc, rcsg_stats* stats, bool sync) {
    if (groups.empty()) throw Failure{RCSG_ERR_CONFIG, "group count must be >= 1"};
    if (slice_end <= slice_begin) throw Failure{RCSG_ERR_CONFIG, "empty slice range"};
    // (re)bind the program to this group list: chunk capacity, arena, chunk
    // index tables.  Repeated calls with the same groups (one call per slice
    // range) reuse everything.
    if (!tree_fixed_) {
        tree_fixed_ = true;
        retree(groups);
    }
    if (precision_ == RCSG_PREC_F16 && !calibrated_)
        calibrate(groups, configs.empty() ? 0 : configs[0], slice_begin);
    if (groups != bound_groups_) bind_groups(groups);
    const int64_t P = nodes_[root_].payload;
    const int64_t acc_n = static_cast<int64_t>(groups.size()) * P * 2;
    try {
        run_bound(groups.size(), configs, slice_begin, slice_end, d_acc, stats, P, acc_n, sync || profile_);
    } catch (const Failure& f) {
        // fp16: an unstorable value means the calibrated scales (first slice, <= 16
        // groups, 2^6 headroom) were too tight for this data, not a non-finite
        // amplitude.  Widen every intermediate's headroom by 2^8, rebind (graph,
        // caches, tables) and rerun; a synchronous call has not touched d_acc.
        if (f.code != RCSG_ERR_NUMERIC || precision_ != RCSG_PREC_F16 || !(sync || profile_) || f16_widened_ >= 3)
            throw;
        ++f16_widened_;
        for (const StepInfo& st : steps_) node_exp_[st.r] += 8;
        bound_groups_.clear();
        run(groups, configs, slice_begin, slice_end, d_acc, stats, sync);
    }
}

void Program::sync() {
    CUDA_OK(cudaStreamSynchronize(stream_));
    if (!fault_pending_) return;
    fault_pending_ = false;
    int32_t fault = INT_MAX;
    CUDA_OK(cudaMemcpy(&fault, d_fault_, sizeof(int32_t), cudaMemcpyDeviceToHost));
    if (fault != INT_MAX)
        throw Failure{RCSG_ERR_NUMERIC, "non-finite intermediate at contraction step " + std::to_string(fault), fault};
}

rcsg_network_desc Program::stored_net() {
    rcsg_network_desc net = calib_net_;
    net.leaf_rank = c_rank_.data();
    net.leaf_labels = c_labels_.data();
    net.leaf_data = leaf_data_.data();
    net.output_labels = c_out_.data();
    net.open_labels = c_openl_.data();
    net.open_qubits = c_openq_.data();
    return net;
}

rcsg_plan_desc Program::stored_plan() {
    rcsg_plan_desc plan = calib_plan_;
    plan.steps = c_steps_.data();
    plan.n_steps = static_cast<int32_t>(c_steps_.size() / 3);
    plan.sliced = c_sliced_.data();
    plan.broken = c_broken_.data();
    plan.fixed_outputs = c_fixed_.data();
    return plan;
}

// First run: reassociate the tree for this group batch (see reassociate()),
// then rebuild the program from the rotated steps.  RCSG_TREE=plan keeps the
// plan's tree as given.
// First run: reassociate the tree for this group batch (see reassociate()),
// then rebuild the program from the rotated steps.  RCSG_TREE=plan keeps the
// plan's tree.
void Program::retree(const std::vector<uint64_t>& groups) {
    const uint64_t plan_flops = plan_flops_;  // stats report the plan's (reference-equivalent) FLOPs
    auto rebuild_program = [&] {
        const rcsg_network_desc net = stored_net();
        const rcsg_plan_desc plan = stored_plan();
        build_nodes(net, plan);
        build_steps();
        plan_flops_ = plan_flops;
        node_exp_.assign(nodes_.size(), 0);
        CUDA_OK(cudaMemcpy(d_canon_, root_canon_src_.data(), root_canon_src_.size() * sizeof(int32_t),
                           cudaMemcpyHostToDevice));
    };
    const char* env = getenv("RCSG_TREE");
    if (env && std::string(env) == "plan") return;
    const int n_steps = static_cast<int>(c_steps_.size() / 3);
    if (n_steps < 2) return;
    std::vector<TreeNode> t(nodes_.size());
    double max_elems = 1;
    std::vector<uint64_t> uniq = groups;
    std::sort(uniq.begin(), uniq.end());
    uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
    double pf = precision_ >= RCSG_PREC_BF16 ? 1.2e15
                : (precision_ == RCSG_PREC_TF32 ? 6e14 : (precision_ == RCSG_PREC_3XTF32 ? 2e14 : 5e13));
    double bw = 6e12, lat = 4e-6;
    if (const char* e = getenv("RCSG_TREE_PF")) pf = atof(e);  // cost-model knobs (experiments)
    if (const char* e = getenv("RCSG_TREE_BW")) bw = atof(e);
    if (const char* e = getenv("RCSG_TREE_LAT")) lat = atof(e);
    TreeCost cost{uniq, pf, bw, static_cast<double>(elem_bytes_), lat, {}};
    for (int i = 0; i < n_leaves_; ++i) {
        t[i].labels = nodes_[i].labels;
        std::sort(t[i].labels.begin(), t[i].labels.end());
        t[i].mask = nodes_[i].var_mask;
        t[i].level = nodes_[i].level;
    }
    for (int s = 0; s < n_steps; ++s) {
        const int r = c_steps_[3 * s + 2];
        t[r].a = c_steps_[3 * s];
        t[r].b = c_steps_[3 * s + 1];
        combine(t, r);
        max_elems = std::max(max_elems, cost.nvar(t[r].mask) * std::ldexp(1.0, static_cast<int>(t[r].labels.size())));
    }
    std::vector<int32_t> steps = c_steps_;
    std::vector<int32_t> origin(n_steps);
    std::iota(origin.begin(), origin.end(), 0);
    const int rot = reassociate(t, steps, origin, cost, max_elems);
    if (getenv("RCSG_DUMP_TREE")) fprintf(stderr, "[rcsg] reassociation: %d rotations\n", rot);
    if (!rot) return;
    c_steps_ = steps;
    step_origin_ = origin;
    rebuild_program();
}

// fp16 mode: per-tensor power-of-two scales.  A transient tf32 program runs one
// pass (first slice, first configuration, up to 16 of the groups) and records
// every node's max |value|; node r is then stored times 2^-e_r with
// e_r = ceil(log2 max_r) - 10, i.e. at most 2^10 in magnitude (64x headroom
// below the fp16 maximum for other slices and groups).  Each GEMM multiplies
// its fp32 result by 2^(e_a + e_b - e_r) before rounding to fp16; finalize
// multiplies the root by 2^e_root.
void Program::calibrate(const std::vector<uint64_t>& groups, uint64_t config, uint64_t slice) {
    rcsg_network_desc net = stored_net();
    rcsg_plan_desc plan = stored_plan();
    // calibration sample: up to 64 groups spread over the caller's list and up
    // to 4 slices spread over the plan's slice range (the call's first slice
    // included); each node's scale covers the max over all of them
    std::vector<uint64_t> sub;
    const size_t n_sub = std::min<size_t>(groups.size(), 64);
    for (size_t i = 0; i < n_sub; ++i) sub.push_back(groups[i * groups.size() / n_sub]);
    std::vector<uint64_t> cal_slices{slice};
    const uint64_t n_slices = uint64_t{1} << calib_plan_.n_sliced;
    for (uint64_t q = 1; q < 4 && q < n_slices; ++q) {
        const uint64_t s = (slice + q * (n_slices / 4 ? n_slices / 4 : 1)) % n_slices;
        if (std::find(cal_slices.begin(), cal_slices.end(), s) == cal_slices.end()) cal_slices.push_back(s);
    }
    std::vector<float> mx(nodes_.size(), 0.f);
    {
        size_t fr = 0, tot = 0;
        CUDA_OK(cudaMemGetInfo(&fr, &tot));
        // (the fp16 arena is allocated after calibration, by the first bind)
        Program cal(net, plan, roles_, RCSG_PREC_TF32, static_cast<uint64_t>(fr * 0.8));
        cal.tree_fixed_ = true;  // the steps are already this program's (reassociated) tree
        cal.step_origin_ = step_origin_;
        CUDA_OK(cudaMalloc(&cal.d_max_, nodes_.size() * sizeof(float)));
        CUDA_OK(cudaMemsetAsync(cal.d_max_, 0, nodes_.size() * sizeof(float), cal.stream()));
        cal.record_max_ = true;
        double* d_acc = nullptr;
        CUDA_OK(cudaMalloc(&d_acc, sub.size() * (size_t{1} << out_rank_) * 2 * sizeof(double)));
        CUDA_OK(cudaMemsetAsync(d_acc, 0, sub.size() * (size_t{1} << out_rank_) * 2 * sizeof(double), cal.stream()));
        std::vector<uint64_t> cfg;
        if (calib_plan_.n_broken) cfg.push_back(config);
        try {
            for (uint64_t s : cal_slices) cal.run(sub, cfg, s, s + 1, d_acc, nullptr);
        } catch (...) {
            cudaFree(d_acc);
            cudaFree(cal.d_max_);
            cal.d_max_ = nullptr;
            throw;
        }
        CUDA_OK(cudaMemcpy(mx.data(), cal.d_max_, mx.size() * sizeof(float), cudaMemcpyDeviceToHost));
        cudaFree(d_acc);
        cudaFree(cal.d_max_);
        cal.d_max_ = nullptr;
    }
    // RCSG_F16_BIAS (test knob): added to every calibrated exponent (negative = tighter)
    const int bias = getenv("RCSG_F16_BIAS") ? atoi(getenv("RCSG_F16_BIAS")) : 0;
    for (const StepInfo& st : steps_) {
        const float m = mx[st.r];
        node_exp_[st.r] = m > 0.f && std::isfinite(m) ? static_cast<int>(std::ceil(std::log2(m))) - 10 + bias
                                                      : node_exp_[st.a] + node_exp_[st.b];
    }
    calibrated_ = true;
    reset_graph();
}

void Program::bind_groups(const std::vector<uint64_t>& groups) {
    n_ext_groups_ = groups.size();
    bound_groups_.clear();
    level0_valid_ = false;
    phase3_valid_ = false;
    tables_valid_ = false;
    reset_graph();
    // chunk capacity: the largest group chunk whose arena fits the budget
    std::vector<uint64_t> uniq = groups;
    std::sort(uniq.begin(), uniq.end());
    uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
    uint64_t budget = mem_budget_;
    if (!budget) {
        size_t fr = 0, tot = 0;
        CUDA_OK(cudaMemGetInfo(&fr, &tot));
        // 3xtf32 stages the hi / lo halves of a GEMM's operands in a workspace next to the arena
        budget = static_cast<uint64_t>(fr * (precision_ == RCSG_PREC_3XTF32 ? 0.3 : 0.7));
    }
    const int64_t n_uniq = static_cast<int64_t>(uniq.size());
    plan_codes_ = n_uniq;
    mark_tables();  // the arena plan keeps the tables' boundary nodes from pass start
    int64_t lo = 1, hi = n_uniq;
    if (static_cast<uint64_t>(plan_arena(1, false)) * elem_bytes_ > budget)
        throw Failure{RCSG_ERR_CAPACITY, "device arena for one group (" +
                                             std::to_string(plan_arena(1, false) * elem_bytes_) +
                                             " B) exceeds the memory budget"};
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) / 2;
        if (static_cast<uint64_t>(plan_arena(mid, false)) * elem_bytes_ <= budget) lo = mid;
        else hi = mid - 1;
    }
    const int64_t cap = lo;
    const int64_t need = plan_arena(cap, true);
    if (need > arena_elems_) {
        cudaFree(arena_);
        arena_ = nullptr;
        CUDA_OK(cudaMalloc(&arena_, static_cast<size_t>(need) * elem_bytes_));
        arena_elems_ = need;
    }
    // static leaf jobs (offsets depend on the arena plan)
    for (int level = 0; level < 2; ++level) {
        static_jobs_[level].clear();
        for (int i = 0; i < n_leaves_; ++i) {
            const NodeInfo& nd = nodes_[i];
            if (nd.level != level) continue;
            LeafJob j{};
            j.out_off = nd.off;
            j.out_plane = nd.plane;
            j.data_off = nd.data_off;
            j.rank = nd.rank0;
            j.out_rank = static_cast<int32_t>(nd.labels.size());
            j.n_var = 1;
            j.codes_off = -1;
            for (int p = 0; p < nd.rank0; ++p) {
                const LabelRole& rl = roles_[nd.labels0[p]];
                j.kind[p] = rl.role;
                j.arg[p] = static_cast<int16_t>(nd.labels0[p]);
                j.obit[p] = rl.role == kFree ? static_cast<int8_t>(nd.labels.size() - 1 - pos_in(nd.labels, nd.labels0[p])) : 0;
            }
            static_jobs_[level].push_back(j);
        }
        cudaFree(d_static_jobs_[level]);
        d_static_jobs_[level] = nullptr;
        CUDA_OK(cudaMalloc(&d_static_jobs_[level], std::max<size_t>(static_jobs_[level].size(), 1) * sizeof(LeafJob)));
        CUDA_OK(cudaMemcpy(d_static_jobs_[level], static_jobs_[level].data(),
                           static_jobs_[level].size() * sizeof(LeafJob), cudaMemcpyHostToDevice));
    }
    prepare_chunks(groups, cap);
    plan_tables();
    build_tasks();
    chunk_cap_ = cap;
    bound_groups_ = groups;
}

// One (configuration, slice) pass after set_pass: level-1 steps, then every
// group chunk's level-2 steps and finalisation.  Replayed as a CUDA graph once
// the first pass has sized the workspaces (every pass launches the same
// kernels; the slice / configuration bits are read from device memory).
void Program::exec_pass_body(int64_t P) {
    exec_phase(1, nullptr);
    for (const ChunkData& ch : chunks_) {
        if (chunks_.size() > 1) exec_phase(3, &ch);  // one chunk: cached outside the pass
        exec_phase(2, &ch);
        const NodeInfo& root = nodes_[root_];
        RCSG_DISPATCH(precision_,
                      launch_finalize<S>(static_cast<const S*>(buf(root.off)), root.plane,
                                         std::ldexp(1.0, node_exp_[root_]), P,
                                         static_cast<int>(root.labels.size()), d_canon_,
                                         static_cast<int>(ch.fin_g.size()), ch.d_fin, ch.d_fin + ch.fin_g.size(),
                                         ch.d_fin + 2 * ch.fin_g.size() + 1,
                                         ch.d_fin + 2 * ch.fin_g.size() + 1 + ch.ent_vid.size(), d_state_, d_part_,
                                         ls_));
        ++launches_;
    }
}

void Program::free_tasks() {
    for (cudaEvent_t e : task_ev_) cudaEventDestroy(e);
    task_ev_.clear();
    tasks_.clear();
    task_wait_.clear();
    task_lane_.clear();
}

// The pass body as tasks in program order, each with the arena regions it
// reads and writes; task u must precede t when t writes memory u reads or
// writes, or reads memory u writes.  Tasks go to kLanes streams (a dependency
// chain stays on one lane); t waits only for the latest dependency per other
// lane.  Same-lane order also serialises the per-stream split-K workspace.
void Program::build_tasks() {
    free_tasks();
    constexpr int kLanes = 8;
    using Region = std::pair<int64_t, int64_t>;
    std::vector<std::vector<Region>> rd, wr;
    auto node_region = [&](int id) { return Region{nodes_[id].off, nodes_[id].off + 2 * nodes_[id].plane}; };
    auto add = [&](Task t, std::vector<Region> r, std::vector<Region> w) {
        tasks_.push_back(t);
        rd.push_back(std::move(r));
        wr.push_back(std::move(w));
    };
    auto leaf_regions = [&](int phase) {
        std::vector<Region> w;
        for (int i = 0; i < n_leaves_; ++i) {
            const NodeInfo& nd = nodes_[i];
            if ((nd.level < 2 ? nd.level : (nd.pass_dep ? 2 : 3)) == phase) w.push_back(node_region(i));
        }
        return w;
    };
    auto add_steps = [&](int phase, const ChunkData* ch) {
        for (const StepInfo& st : steps_) {
            if (st.phase != phase || st.tab) continue;
            std::vector<Region> r{node_region(st.a), node_region(st.b)}, w{node_region(st.r)};
            if (st.perm_a) w.push_back({st.sa_off, st.sa_off + 2 * st.sa_plane});
            if (st.perm_b) w.push_back({st.sb_off, st.sb_off + 2 * st.sb_plane});
            add({1, &st, ch}, r, w);
        }
    };
    const Region part{-2, -1};  // the per-configuration accumulator
    if (!static_jobs_[1].empty()) add({0, nullptr, nullptr}, {}, leaf_regions(1));
    if (!tab_jobs_.empty()) {
        std::vector<Region> w;
        for (const TableJob& j : tab_jobs_) w.push_back({j.node_off, j.node_off + 2 * j.node_plane});
        add({6, nullptr, nullptr}, {}, w);
    }
    add_steps(1, nullptr);
    for (const ChunkData& ch : chunks_) {
        if (chunks_.size() > 1) {  // one chunk: phase 3 is cached outside the pass
            if (ch.n_leaf_jobs3) add({4, nullptr, &ch}, {}, leaf_regions(3));
            add_steps(3, &ch);
        }
        if (ch.n_leaf_jobs > ch.n_leaf_jobs3) add({2, nullptr, &ch}, {}, leaf_regions(2));
        add_steps(2, &ch);
        add({3, nullptr, &ch}, {node_region(root_)}, {part});
    }
    const int T = static_cast<int>(tasks_.size());
    auto overlap = [](const std::vector<Region>& x, const std::vector<Region>& y) {
        for (const Region& a : x)
            for (const Region& b : y)
                if (a.first < b.second && b.first < a.second) return true;
        return false;
    };
    std::vector<int> tail(kLanes, -1);
    task_lane_.assign(T, 0);
    task_wait_.assign(T, {});
    n_lanes_used_ = 1;
    for (int t = 0; t < T; ++t) {
        std::vector<int> deps;
        for (int u = 0; u < t; ++u)
            if (overlap(wr[t], rd[u]) || overlap(wr[t], wr[u]) || overlap(rd[t], wr[u])) deps.push_back(u);
        int lane = -1;
        for (auto it = deps.rbegin(); it != deps.rend() && lane < 0; ++it)
            for (int l = 0; l < kLanes; ++l)
                if (tail[l] == *it) lane = l;
        if (lane < 0) {  // the least recently used lane
            lane = 0;
            for (int l = 1; l < kLanes; ++l)
                if (tail[l] < tail[lane]) lane = l;
        }
        task_lane_[t] = lane;
        tail[lane] = t;
        n_lanes_used_ = std::max(n_lanes_used_, lane + 1);
        std::vector<int> last(kLanes, -1);
        for (int u : deps)
            if (task_lane_[u] != lane) last[task_lane_[u]] = std::max(last[task_lane_[u]], u);
        for (int l = 0; l < kLanes; ++l)
            if (last[l] >= 0) task_wait_[t].push_back(last[l]);
    }
    if (getenv("RCSG_DUMP_TREE")) {  // longest dependency chain, in tasks
        std::vector<int> depth(T, 1);
        int longest = 0;
        for (int t = 0; t < T; ++t) {
            for (int u = 0; u < t; ++u)
                if (overlap(wr[t], rd[u]) || overlap(wr[t], wr[u]) || overlap(rd[t], wr[u]))
                    depth[t] = std::max(depth[t], depth[u] + 1);
            longest = std::max(longest, depth[t]);
        }
        fprintf(stderr, "[rcsg] pass DAG: %d tasks on %d lanes, longest chain %d\n", T, n_lanes_used_, longest);
        for (int t = 0; t < T; ++t) {
            const Task& k = tasks_[t];
            if (k.kind != 1) {
                fprintf(stderr, "  task %3d kind %d depth %d\n", t, k.kind, depth[t]);
                continue;
            }
            const StepInfo& st = *k.st;
            auto nv = [&](int id) -> long long {
                return (nodes_[id].level == 2 && k.ch) ? (long long)k.ch->nvar[id] : 1LL;
            };
            fprintf(stderr, "  task %3d step %4d L%d mode %d m %lld n %lld k %lld va %lld vb %lld vr %lld macs %.3g depth %d\n",
                    t, st.plan_index, st.level, st.mode, (long long)st.m, (long long)st.n, (long long)st.k,
                    nv(st.a), nv(st.b), nv(st.r), (double)st.m * st.n * st.k * (st.mode == 1 ? nv(st.a) : nv(st.r)),
                    depth[t]);
        }
    }
    task_ev_.resize(T);
    for (int t = 0; t < T; ++t) CUDA_OK(cudaEventCreateWithFlags(&task_ev_[t], cudaEventDisableTiming));
    while (static_cast<int>(lanes_.size()) < n_lanes_used_) {
        cudaStream_t l;
        CUDA_OK(cudaStreamCreateWithFlags(&l, cudaStreamNonBlocking));
        lanes_.push_back(l);
    }
    while (static_cast<int>(lane_ev_.size()) < n_lanes_used_ + 1) {
        cudaEvent_t e;
        CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        lane_ev_.push_back(e);
    }
}

// Slice tables.  A per-pass step is tabulated when its result is small, does
// not depend on the configuration, and each operand is a leaf, a constant node
// or itself tabulated.  Boundary nodes (tabulated, consumed by a per-pass
// step) get a table over the sliced labels in their subtree; the tables are
// filled once per binding by evaluating the tabulated steps for every value of
// the union of those labels (at most 2^10 evaluations), and each pass gathers
// its entries with one launch.  RCSG_NO_TABLES=1 disables.
void Program::mark_tables() {
    tab_region_mask_ = 0;
    tab_boundary_.clear();
    for (NodeInfo& nd : nodes_) nd.tab = false;
    for (StepInfo& st : steps_) st.tab = false;
    if (getenv("RCSG_NO_TABLES") || record_max_) return;
    constexpr int64_t kTabMaxPayload = int64_t{1} << 16;
    auto usable = [&](int id) {
        const NodeInfo& nd = nodes_[id];
        return nd.is_leaf ? nd.level < 2 : (nd.level == 0 || nd.tab);
    };
    for (StepInfo& st : steps_) {
        NodeInfo& R = nodes_[st.r];
        if (st.phase != 1 || R.cfg_dep || R.payload > kTabMaxPayload || !usable(st.a) || !usable(st.b)) continue;
        st.tab = R.tab = true;
    }
    std::vector<int>& boundary = tab_boundary_;
    for (const StepInfo& st : steps_) {
        if (!st.tab) continue;
        const int c = nodes_[st.r].consumer;
        bool consumed_by_tab = false;
        for (const StepInfo& s2 : steps_)
            if (c >= 0 && (&s2 - steps_.data()) == c) consumed_by_tab = s2.tab;
        if (!consumed_by_tab) {
            boundary.push_back(st.r);
            tab_region_mask_ |= nodes_[st.r].slice_mask;
        }
    }
    if (boundary.empty() || __builtin_popcountll(tab_region_mask_) > 10) {  // too many evaluations
        for (NodeInfo& nd : nodes_) nd.tab = false;
        for (StepInfo& st : steps_) st.tab = false;
        tab_region_mask_ = 0;
        boundary.clear();
    }
}

// tables and gather jobs of the marked boundary nodes (arena offsets assigned)
void Program::plan_tables() {
    for (void* t : tab_mem_) cudaFree(t);
    tab_mem_.clear();
    cudaFree(d_tab_jobs_);
    d_tab_jobs_ = nullptr;
    tab_jobs_.clear();
    const std::vector<int>& boundary = tab_boundary_;
    if (boundary.empty()) return;
    for (int id : boundary) {
        const NodeInfo& nd = nodes_[id];
        TableJob j{};
        j.node_off = nd.off;
        j.node_plane = nd.plane;
        j.payload = nd.payload;
        j.mask = nd.slice_mask;
        const size_t bytes = (size_t{1} << __builtin_popcountll(j.mask)) * 2 * nd.payload * elem_bytes_;
        CUDA_OK(cudaMalloc(&j.table, std::max<size_t>(bytes, 16)));
        tab_mem_.push_back(j.table);
        tab_jobs_.push_back(j);
    }
    CUDA_OK(cudaMalloc(&d_tab_jobs_, tab_jobs_.size() * sizeof(TableJob)));
    CUDA_OK(cudaMemcpy(d_tab_jobs_, tab_jobs_.data(), tab_jobs_.size() * sizeof(TableJob), cudaMemcpyHostToDevice));
    if (getenv("RCSG_DUMP_TREE")) {
        int n_tab = 0;
        for (const StepInfo& st : steps_) n_tab += st.tab;
        fprintf(stderr, "[rcsg] slice tables: %d tabulated steps, %zu boundary nodes, %d sliced labels\n", n_tab,
                boundary.size(), __builtin_popcountll(tab_region_mask_));
    }
}

void Program::build_tables() {
    const int bits = __builtin_popcountll(tab_region_mask_);
    for (uint64_t combo = 0; combo < (uint64_t{1} << bits); ++combo) {
        uint64_t slice = 0;  // deposit combo onto the region's sliced bits
        int b = 0;
        for (uint64_t m = tab_region_mask_; m; m &= m - 1, ++b)
            if ((combo >> b) & 1) slice |= m & (~m + 1);
        launch_set_pass(d_state_, slice, 0, 0, 1, stream_);
        if (!static_jobs_[1].empty()) {
            RCSG_DISPATCH(precision_, launch_leaf_project<S>(d_static_jobs_[1], static_cast<int>(static_jobs_[1].size()),
                                                            d_leaf_data_, nullptr, d_pass_src_, d_state_,
                                                            static_cast<S*>(arena_), stream_, round_leaves()));
        }
        for (const StepInfo& st : steps_)
            if (st.tab) exec_step(st, nullptr);
        launch_table_io(d_tab_jobs_, static_cast<int>(tab_jobs_.size()), d_state_, arena_, elem_bytes_, 1, stream_);
    }
}

void Program::run_task(const Task& t, int64_t P) {
    switch (t.kind) {
        case 0:
            RCSG_DISPATCH(precision_, launch_leaf_project<S>(d_static_jobs_[1], static_cast<int>(static_jobs_[1].size()),
                                                            d_leaf_data_, nullptr, d_pass_src_, d_state_,
                                                            static_cast<S*>(arena_), ls_, round_leaves()));
            ++launches_;
            break;
        case 1:
            exec_step(*t.st, t.ch);
            break;
        case 6:
            launch_table_io(d_tab_jobs_, static_cast<int>(tab_jobs_.size()), d_state_, arena_, elem_bytes_, 0, ls_);
            ++launches_;
            break;
        case 2:
        case 4: {
            const int j0 = t.kind == 4 ? 0 : t.ch->n_leaf_jobs3;
            const int j1 = t.kind == 4 ? t.ch->n_leaf_jobs3 : t.ch->n_leaf_jobs;
            RCSG_DISPATCH(precision_, launch_leaf_project<S>(t.ch->d_leaf_jobs + j0, j1 - j0, d_leaf_data_,
                                                            t.ch->d_codes, d_pass_src_, d_state_,
                                                            static_cast<S*>(arena_), ls_, round_leaves()));
            ++launches_;
            break;
        }
        default: {
            const NodeInfo& root = nodes_[root_];
            RCSG_DISPATCH(precision_,
                          launch_finalize<S>(static_cast<const S*>(buf(root.off)), root.plane,
                                             std::ldexp(1.0, node_exp_[root_]), P,
                                             static_cast<int>(root.labels.size()), d_canon_,
                                             static_cast<int>(t.ch->fin_g.size()), t.ch->d_fin,
                                             t.ch->d_fin + t.ch->fin_g.size(), t.ch->d_fin + 2 * t.ch->fin_g.size() + 1,
                                             t.ch->d_fin + 2 * t.ch->fin_g.size() + 1 + t.ch->ent_vid.size(), d_state_,
                                             d_part_, ls_));
            ++launches_;
        }
    }
}

// fork from stream_, run the tasks on their lanes, join back into stream_
void Program::exec_pass_dag(int64_t P) {
    CUDA_OK(cudaEventRecord(lane_ev_[0], stream_));
    for (int l = 0; l < n_lanes_used_; ++l) CUDA_OK(cudaStreamWaitEvent(lanes_[l], lane_ev_[0], 0));
    for (size_t t = 0; t < tasks_.size(); ++t) {
        ls_ = lanes_[task_lane_[t]];
        for (int u : task_wait_[t]) CUDA_OK(cudaStreamWaitEvent(ls_, task_ev_[u], 0));
        run_task(tasks_[t], P);
        CUDA_OK(cudaEventRecord(task_ev_[t], ls_));
    }
    ls_ = stream_;
    for (int l = 0; l < n_lanes_used_; ++l) {
        CUDA_OK(cudaEventRecord(lane_ev_[l + 1], lanes_[l]));
        CUDA_OK(cudaStreamWaitEvent(stream_, lane_ev_[l + 1], 0));
    }
}

void Program::reset_graph() {
    if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
    graph_exec_ = nullptr;
    graph_warm_ = false;
}

void Program::run_pass_body(int64_t P) {
    static const bool no_graph = getenv("RCSG_NO_GRAPH") != nullptr;
    if (profile_ || no_graph) {
        exec_pass_body(P);
        return;
    }
    static const bool no_dag = getenv("RCSG_NO_DAG") != nullptr;
    if (!graph_exec_ && !graph_warm_) {  // first pass: eager, sizes the lanes' split-K workspaces
        if (no_dag) exec_pass_body(P);
        else exec_pass_dag(P);
        graph_warm_ = true;
        return;
    }
    if (!graph_exec_) {
        const uint64_t before = launches_, flops_before = exec_flops_;
        cudaGraph_t graph;
        CUDA_OK(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
        if (no_dag) exec_pass_body(P);
        else exec_pass_dag(P);
        CUDA_OK(cudaStreamEndCapture(stream_, &graph));
        CUDA_OK(cudaGraphInstantiate(&graph_exec_, graph, 0));
        cudaGraphDestroy(graph);
        graph_launches_ = launches_ - before;
        graph_flops_ = exec_flops_ - flops_before;
        launches_ = before;
        exec_flops_ = flops_before;
    }
    CUDA_OK(cudaGraphLaunch(graph_exec_, stream_));
    launches_ += graph_launches_;
    exec_flops_ += graph_flops_;
}

void Program::run_bound(size_t n_groups, const std::vector<uint64_t>& configs, uint64_t slice_begin,
                        uint64_t slice_end, double* d_acc, rcsg_stats* stats, int64_t P, int64_t acc_n,
                        bool sync) {
    if (acc_n > acc_cap_) {
        cudaFree(d_part_);
        cudaFree(d_res_);
        cudaFree(d_comp_);
        reset_graph();
        CUDA_OK(cudaMalloc(&d_part_, acc_n * sizeof(double)));
        CUDA_OK(cudaMalloc(&d_res_, acc_n * sizeof(double)));
        CUDA_OK(cudaMalloc(&d_comp_, acc_n * sizeof(double)));
        acc_cap_ = acc_n;
    }
    if (!fault_pending_) {  // the flag still holds an unchecked async run's fault otherwise
        static const int32_t no_fault = INT_MAX;
        CUDA_OK(cudaMemcpyAsync(d_fault_, &no_fault, sizeof(int32_t), cudaMemcpyHostToDevice, stream_));
    }
    launch_fill(d_res_, 0.0, acc_n, stream_);
    launch_fill(d_comp_, 0.0, acc_n, stream_);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (sync) {
        CUDA_OK(cudaEventCreate(&e0));
        CUDA_OK(cudaEventCreate(&e1));
        CUDA_OK(cudaEventRecord(e0, stream_));
    }
    launches_ = 0;
    exec_flops_ = 0;
    uint64_t passes = 0;
    const std::vector<uint64_t> no_cfg{0};
    const std::vector<uint64_t>& cfgs = configs.empty() ? no_cfg : configs;
    // level 0 depends on no slice, configuration or group: computed once per
    // arena binding and kept (its results persist in the arena across calls)
    if (!level0_valid_) {
        launch_set_pass(d_state_, slice_begin, cfgs[0], 0, 1, stream_);
        exec_phase(0, nullptr);
        level0_valid_ = true;
    }
    if (!phase3_valid_ && chunks_.size() == 1) {  // group-only results of the single chunk
        exec_phase(3, &chunks_[0]);
        phase3_valid_ = true;
    }
    if (!tables_valid_ && !tab_jobs_.empty()) {
        build_tables();
        tables_valid_ = true;
    }
    for (size_t ci = 0; ci < cfgs.size(); ++ci) {
        launch_fill(d_part_, 0.0, acc_n, stream_);
        ++launches_;
        for (uint64_t s = slice_begin; s < slice_end; ++s) {  // slices ascending
            launch_set_pass(d_state_, s, cfgs[ci], 0, 1, stream_);
            ++launches_;
            run_pass_body(P);
            passes += chunks_.size();
        }
        launch_kahan(d_res_, d_comp_, d_part_, acc_n, stream_);
        ++launches_;
    }
    if (sync) {  // a fault must surface before the caller's buffer is touched (fp16 retry)
        CUDA_OK(cudaStreamSynchronize(stream_));
        int32_t fault = INT_MAX;
        CUDA_OK(cudaMemcpy(&fault, d_fault_, sizeof(int32_t), cudaMemcpyDeviceToHost));
        if (fault != INT_MAX) {
            fault_pending_ = false;
            throw Failure{RCSG_ERR_NUMERIC, "non-finite intermediate at contraction step " + std::to_string(fault),
                          fault};
        }
    }
    // d_acc += res
    launch_fill(d_comp_, 0.0, acc_n, stream_);
    launch_kahan(d_acc, d_comp_, d_res_, acc_n, stream_);
    launches_ += 2;
    float ms = 0;
    CUDA_OK(cudaGetLastError());
    if (sync) {
        CUDA_OK(cudaEventRecord(e1, stream_));
        CUDA_OK(cudaEventSynchronize(e1));
        CUDA_OK(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        collect_marks(stats);
    }
    fault_pending_ = true;
    if (sync) this->sync();
    if (stats) {
        stats->plan_flops += plan_flops_ * static_cast<uint64_t>(n_groups) * cfgs.size() * (slice_end - slice_begin);
        stats->executed_flops += exec_flops_;
        stats->arena_bytes = static_cast<uint64_t>(arena_elems_) * elem_bytes_;
        stats->kernel_launches += launches_;
        stats->passes += passes;
        stats->device_ms += ms;
    }
}

}  // namespace rcsg
