// Sampler API (namespace rcs): candidate sets on the host (bit-identical RNG
// stream, sampling.cpp:14-60), selection / sampling on the GPU (rcsg.h).
#include <algorithm>
#include <cmath>
#include <memory>

#include "rcs_b200.hpp"
#include "rcsg.h"

namespace rcs {
namespace {

[[noreturn]] void raise(int rc) {
    int32_t step = -1;
    const std::string msg = rcsg_last_error(&step);
    if (rc == RCSG_ERR_CONFIG) throw ConfigError(msg);
    if (rc == RCSG_ERR_NUMERIC) throw NumericFault(msg, step);
    if (rc == RCSG_ERR_CAPACITY) throw CapacityError(msg);
    throw DeviceError(msg);
}

// Evaluates the ProbFn over every candidate (g, i) and stages it on the device.
struct DeviceProbs {
    void* d = nullptr;
    DeviceProbs(const CandidateSet& cs, const ProbFn& p) {
        const std::uint64_t per = std::uint64_t{1} << cs.l();
        std::vector<double> h(cs.size());
        for (std::uint64_t g = 0; g < cs.n_groups(); ++g)
            for (std::uint64_t i = 0; i < per; ++i) h[g * per + i] = p(cs.member(g, i));
        if (int rc = rcsg_device_alloc(h.size() * sizeof(double), &d)) raise(rc);
        if (int rc = rcsg_memcpy(d, h.data(), h.size() * sizeof(double), 1)) raise(rc);
    }
    ~DeviceProbs() {
        if (d) rcsg_device_free(d);
    }
};

rcsg_candidates describe(const CandidateSet& cs) {
    return rcsg_candidates{cs.n_qubits, cs.l(), cs.open_qubits.data(), cs.n_groups(), cs.group_fixed.data()};
}

}  // namespace

std::uint64_t CandidateSet::member(std::uint64_t group, std::uint64_t i) const {
    std::uint64_t index = 0;
    for (int j = 0; j < l(); ++j) index |= ((i >> j) & 1ull) << open_qubits[j];
    const std::uint64_t fixed = group_fixed[group];
    int b = 0, j = 0;
    for (int q = 0; q < n_qubits; ++q) {
        if (j < l() && open_qubits[j] == q) {
            ++j;
            continue;
        }
        index |= ((fixed >> b++) & 1ull) << q;
    }
    return index;
}

CandidateSet build_candidate_set(int n_qubits, std::vector<int> open_qubits, std::uint64_t n_groups,
                                 std::uint64_t seed) {
    std::sort(open_qubits.begin(), open_qubits.end());
    if (std::adjacent_find(open_qubits.begin(), open_qubits.end()) != open_qubits.end())
        throw ConfigError("open qubits must be distinct");
    for (int q : open_qubits)
        if (q < 0 || q >= n_qubits) throw ConfigError("open qubit out of range");
    const int l = static_cast<int>(open_qubits.size());
    if (n_groups < 1) throw ConfigError("group count must be >= 1");
    if (l == n_qubits && n_groups > 1)
        throw ConfigError("all qubits open: group count must be 1 (groups would collide)");
    CandidateSet cs;
    cs.n_qubits = n_qubits;
    cs.open_qubits = std::move(open_qubits);
    const int n_fixed = n_qubits - l;
    if (n_fixed == 0) {
        cs.group_fixed.push_back(0);
        return cs;
    }
    Rng rng(seed);
    cs.group_fixed.reserve(n_groups);
    for (std::uint64_t g = 0; g < n_groups; ++g) cs.group_fixed.push_back(rng.next_below(std::uint64_t{1} << n_fixed));
    std::vector<std::uint64_t> s = cs.group_fixed;
    std::sort(s.begin(), s.end());
    for (std::size_t i = 1; i < s.size(); ++i) cs.duplicate_groups += s[i] == s[i - 1];
    return cs;
}

double xeb(const SampleSet& samples, const ProbFn& q) {
    std::vector<double> qs;
    qs.reserve(samples.bitstrings.size());
    for (std::uint64_t s : samples.bitstrings) qs.push_back(q(s));
    double out = 0;
    if (int rc = rcsg_xeb(samples.n_qubits, qs.size(), qs.data(), &out)) raise(rc);
    return out;
}

std::uint64_t lexicographic_key(std::uint64_t index, int n_qubits) {
    std::uint64_t key = 0;
    for (int q = 0; q < n_qubits; ++q) key |= ((index >> q) & 1ull) << (n_qubits - 1 - q);
    return key;
}

SampleSet top_k_select(const CandidateSet& candidates, const ProbFn& p, std::uint64_t k) {
    if (k < 1 || k > candidates.size())
        throw ConfigError("top-k size k=" + std::to_string(k) + " outside [1, " +
                          std::to_string(candidates.size()) + "]");
    DeviceProbs dp(candidates, p);
    const rcsg_candidates d = describe(candidates);
    SampleSet out;
    out.n_qubits = candidates.n_qubits;
    out.provenance = Provenance::TopK;
    out.k = k;
    out.bitstrings.resize(k);
    if (int rc = rcsg_topk_probs(&d, static_cast<const double*>(dp.d), k, out.bitstrings.data())) raise(rc);
    return out;
}

SampleSet direct_sample(const CandidateSet& candidates, const ProbFn& p, std::uint64_t rng_seed) {
    DeviceProbs dp(candidates, p);
    const rcsg_candidates d = describe(candidates);
    SampleSet out;
    out.n_qubits = candidates.n_qubits;
    out.provenance = Provenance::Direct;
    out.bitstrings.resize(candidates.n_groups());
    if (int rc = rcsg_direct_sample_probs(&d, static_cast<const double*>(dp.d), rng_seed, out.bitstrings.data()))
        raise(rc);
    return out;
}

double predicted_topk_xeb(double fidelity, std::uint64_t candidate_size, std::uint64_t k) {
    if (fidelity < 0.0 || fidelity > 1.0) throw ConfigError("fidelity outside [0, 1]");
    if (k < 1 || k > candidate_size) throw ConfigError("k outside [1, candidate_size]");
    return fidelity * std::log(static_cast<double>(candidate_size) / static_cast<double>(k));
}

}  // namespace rcs
