// GPU checks of the C++ drop-in API (include/rcs_b200.hpp), run by
// tests/test_gpu_cpp_api.py:
//   1. program cache: 64 contract_group calls (the reference's per-group loop,
//      contraction_engine.cpp:307-325) against one contract_groups call;
//   2. device context: contract(..., workers) sharded over 1 and 2 GPUs is
//      bit-identical (test_contraction.cpp:84-93), and matches the one-GPU
//      unsharded contract() to rounding.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <map>

#include "rcs_b200.hpp"

using clk = std::chrono::steady_clock;

static double rel(const std::vector<rcs::cplx>& a, const std::vector<rcs::cplx>& b) {
    double num = 0, den = 0;
    for (std::size_t i = 0; i < a.size(); ++i) {
        num += std::norm(a[i] - b[i]);
        den += std::norm(b[i]);
    }
    return std::sqrt(num / (den > 0 ? den : 1e-300));
}

int main(int argc, char** argv) {
    const int n_gpus = argc > 1 ? std::atoi(argv[1]) : 1;
    rcs::set_precision("f64");
    {
        const auto circ = rcs::gen_random_circuit(12, 8, "grid(3,4)", 1);
        const auto net = rcs::circuit_to_network(circ, {0, 1, 2});
        const auto plan = rcs::find_contraction_path(net, 1ull << 30, rcs::SearchEffort::Low, 1);
        const auto cs = rcs::build_candidate_set(12, {0, 1, 2}, 64, rcs::Rng(1).split(0xca11d).next_u64());
        auto t0 = clk::now();
        rcs::contract_groups(net, plan, nullptr, cs.group_fixed);  // compile + bind (cached afterwards)
        const double t_compile = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
        rcs::contract_group(net, plan, nullptr, 0, cs.group_fixed[0]);
        t0 = clk::now();
        const auto batch = rcs::contract_groups(net, plan, nullptr, cs.group_fixed);
        const double t_batch = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
        t0 = clk::now();
        double worst = 0;
        for (std::size_t g = 0; g < cs.group_fixed.size(); ++g) {
            const auto one = rcs::contract_group(net, plan, nullptr, g, cs.group_fixed[g]);
            worst = std::max(worst, rel(one.amplitudes, batch[g].amplitudes));
        }
        const double t_loop = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
        std::printf("cache compile_ms %.3f batch_ms %.3f loop64_ms %.3f worst_rel %.3e\n", t_compile, t_batch, t_loop,
                    worst);
    }
    {
        rcs::set_precision("tf32");
        const auto circ = rcs::gen_random_circuit(53, 6, "sycamore53", 1);
        const auto net = rcs::circuit_to_network(circ, {0, 1, 2, 3, 4, 5});
        const auto plan = rcs::find_contraction_path(net, 1ull << 20, rcs::SearchEffort::Low, 1);
        std::map<rcs::Label, int> fixed;  // group 0b1011...: every non-open output pinned
        int b = 0;
        for (int q = 6; q < 53; ++q, ++b) fixed[net.output_labels[q]] = (0x5a5a5a5a5a5aull >> b) & 1;
        const auto single = rcs::contract(net, plan, nullptr, fixed, 1).amplitudes;  // no context: one GPU
        rcs::init_devices({0});
        const auto w1 = rcs::contract(net, plan, nullptr, fixed, 1).amplitudes;
        std::printf("multi slices %llu devices1 rel_vs_single %.3e\n",
                    static_cast<unsigned long long>(plan.n_slices()), rel(w1, single));
        if (n_gpus >= 2) {
            rcs::init_devices({0, 1});
            const auto w2 = rcs::contract(net, plan, nullptr, fixed, 2).amplitudes;
            const auto w1b = rcs::contract(net, plan, nullptr, fixed, 1).amplitudes;
            bool same = w2.size() == w1.size();
            for (std::size_t i = 0; same && i < w1.size(); ++i) same = w1[i] == w2[i] && w1[i] == w1b[i];
            std::printf("multi devices2 bit_identical %d rel_vs_single %.3e\n", same ? 1 : 0, rel(w2, single));
        }
        rcs::init_devices({});
    }
    return 0;
}
