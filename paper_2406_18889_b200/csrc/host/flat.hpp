// Flattened (network, plan) descriptors for the C ABI (internal header).
#pragma once
#include <algorithm>
#include <memory>
#include <vector>

#include "rcs_b200.hpp"
#include "rcsg.h"

namespace rcs {

// Flat copies of the network and plan, kept alive with their descriptors.
struct Flat {
    std::vector<int32_t> rank, labels, out_l, open_l, open_q, steps, sliced, broken, fixed;
    std::vector<double> data;
    rcsg_network_desc net{};
    rcsg_plan_desc plan{};
};

inline std::unique_ptr<Flat> flatten(const TensorNetwork& n, const ContractionPlan& p) {
    auto f = std::make_unique<Flat>();
    for (const Tensor& t : n.tensors) {
        if (t.data.size() != (std::size_t{1} << t.labels.size()))
            throw ConfigError("tensor data size does not match its rank");
        f->rank.push_back(t.rank());
        f->labels.insert(f->labels.end(), t.labels.begin(), t.labels.end());
        for (const cplx& v : t.data) {
            f->data.push_back(v.real());
            f->data.push_back(v.imag());
        }
    }
    f->out_l.assign(n.output_labels.begin(), n.output_labels.end());
    // open legs sorted by qubit (canonical order is by ascending qubit)
    std::vector<std::pair<int, int>> oq;
    for (std::size_t i = 0; i < n.open_labels.size(); ++i) oq.push_back({n.open_qubits[i], n.open_labels[i]});
    std::sort(oq.begin(), oq.end());
    for (auto [q, l] : oq) {
        f->open_q.push_back(q);
        f->open_l.push_back(l);
    }
    for (const PlanStep& s : p.steps) {
        f->steps.push_back(s.lhs);
        f->steps.push_back(s.rhs);
        f->steps.push_back(s.result);
    }
    f->sliced.assign(p.sliced.begin(), p.sliced.end());
    f->broken.assign(p.broken.begin(), p.broken.end());
    f->fixed.assign(p.fixed_outputs.begin(), p.fixed_outputs.end());
    f->net = rcsg_network_desc{static_cast<int32_t>(n.tensors.size()), f->rank.data(), f->labels.data(),
                               f->data.data(), static_cast<int32_t>(n.label_names.size()), n.n_qubits,
                               f->out_l.data(), static_cast<int32_t>(f->open_l.size()), f->open_l.data(),
                               f->open_q.data()};
    f->plan = rcsg_plan_desc{static_cast<int32_t>(p.steps.size()), f->steps.data(),
                             static_cast<int32_t>(f->sliced.size()), f->sliced.data(),
                             static_cast<int32_t>(f->broken.size()), f->broken.data(),
                             static_cast<int32_t>(f->fixed.size()), f->fixed.data()};
    return f;
}

}  // namespace rcs
