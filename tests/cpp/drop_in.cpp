// Compile-and-link check of the C++ drop-in API (include/rcs_b200.hpp): the
// calls a reference-side caller makes (harness.cpp:131-152 shape), host-only
// parts, so it runs without a GPU.  Prints a few values the Python test
// compares with the reference library.
#include <cstdio>
#include <sstream>

#include "rcs_b200.hpp"

int main() {
    const auto circ = rcs::gen_random_circuit(30, 14, "grid(5,6)", 1);
    const auto net = rcs::circuit_to_network(circ, {0, 1, 2, 3, 4, 5});
    const auto plan = rcs::find_contraction_path(net, 3ull << 30, rcs::SearchEffort::Low, 1);
    const auto cs = rcs::build_candidate_set(30, {0, 1, 2, 3, 4, 5}, 64, rcs::Rng(1).split(0xca11d).next_u64());
    std::printf("steps %zu sliced %zu flops_per_slice %.17g\n", plan.steps.size(), plan.sliced.size(),
                static_cast<double>(plan.flops_per_slice));
    std::printf("group0 %llu group63 %llu dup %d\n", static_cast<unsigned long long>(cs.group_fixed[0]),
                static_cast<unsigned long long>(cs.group_fixed[63]), cs.duplicate_groups);
    {  // QSVD round trip (reference format)
        rcs::StateVector sv;
        sv.n_qubits = 3;
        for (int i = 0; i < 8; ++i) sv.amps.push_back(rcs::cplx(0.5 * i, -0.25 * i));
        std::stringstream ss;
        rcs::dump_amplitudes(sv, ss);
        const std::string bytes = ss.str();
        const auto back = rcs::load_amplitudes(ss);
        std::printf("qsvd %zu %d %d\n", bytes.size(), back.n_qubits, back.amps == sv.amps ? 1 : 0);
    }
    try {  // device calls raise DeviceError without a GPU (no silent CPU fallback)
        rcs::set_precision("f16");
        auto amps = rcs::contract_group(net, plan, nullptr, 0, cs.group_fixed[0]);
        std::printf("device %zu\n", amps.amplitudes.size());
    } catch (const rcs::DeviceError& e) {
        std::printf("device error\n");
    }
    return 0;
}
