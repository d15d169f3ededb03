// Multi-GPU context of the C ABI (rcsg_init / rcsg_context_* / rcsg_multi_*):
// one host thread drives every listed local GPU; a compiled program per device;
// one NCCL communicator clique over them (ncclCommInitAll, NVLink/NVSwitch).
//
// Slice sharding: the slice range is cut into a fixed number of
// canonical contiguous blocks (independent of the device count); blocks go to
// devices round-robin; each device sums its blocks' slices in ascending order
// into one device partial per block (Program::run, contraction_engine.cpp:241-255
// per block); the partials of the other devices are gathered to the first
// device with NCCL send/recv (the path's only exchange step, kept on the
// device), and that device adds the blocks in block order.  The result is
// therefore bit-identical for 1, 2, 4 or 8 GPUs - the reference's
// worker-count invariance (test_contraction.cpp:84-93).
//
// NCCL is resolved at run time (dlopen of libnccl.so.2: the copy torch already
// loaded, else the system one), so the library has no link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "executor.hpp"
#include "rcsg.h"

using namespace rcsg;

namespace {

#define CUDA_OK(x)                                                                              \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess)                                                                  \
            throw Failure{RCSG_ERR_DEVICE, std::string("CUDA: ") + cudaGetErrorString(e_) + " at " #x}; \
    } while (0)

struct Nccl {
    void* h = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
    static Nccl n = [] {
        Nccl x;
        x.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!x.h) x.h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!x.h) return x;
        x.CommInitAll = reinterpret_cast<decltype(x.CommInitAll)>(dlsym(x.h, "ncclCommInitAll"));
        x.CommDestroy = reinterpret_cast<decltype(x.CommDestroy)>(dlsym(x.h, "ncclCommDestroy"));
        x.GroupStart = reinterpret_cast<decltype(x.GroupStart)>(dlsym(x.h, "ncclGroupStart"));
        x.GroupEnd = reinterpret_cast<decltype(x.GroupEnd)>(dlsym(x.h, "ncclGroupEnd"));
        x.Send = reinterpret_cast<decltype(x.Send)>(dlsym(x.h, "ncclSend"));
        x.Recv = reinterpret_cast<decltype(x.Recv)>(dlsym(x.h, "ncclRecv"));
        x.GetErrorString = reinterpret_cast<decltype(x.GetErrorString)>(dlsym(x.h, "ncclGetErrorString"));
        return x;
    }();
    return n;
}

void nccl_ok(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw Failure{RCSG_ERR_DEVICE, std::string("NCCL: ") + what + ": " +
                                           (nccl().GetErrorString ? nccl().GetErrorString(r) : "error")};
}

// out[i] = sum over b (ascending) of parts[b * n + i]
__global__ void block_sum_kernel(const double* __restrict__ parts, int n_blocks, int64_t n, double* __restrict__ out) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double s = 0.0;
        for (int b = 0; b < n_blocks; ++b) s = __dadd_rn(s, parts[b * n + i]);
        out[i] = s;
    }
}

std::vector<LabelRole> roles_for_groups(const rcsg_network_desc& net, const rcsg_plan_desc& plan) {
    std::vector<LabelRole> roles(net.n_labels);
    std::vector<char> open(net.n_qubits, 0);
    for (int j = 0; j < net.n_open; ++j) {
        if (net.open_qubits[j] < 0 || net.open_qubits[j] >= net.n_qubits)
            throw Failure{RCSG_ERR_CONFIG, "open qubit out of range"};
        open[net.open_qubits[j]] = 1;
    }
    int bit = 0;
    for (int q = 0; q < net.n_qubits; ++q) {
        if (open[q]) continue;
        const int l = net.output_labels[q];
        if (l < 0 || l >= net.n_labels) throw Failure{RCSG_ERR_CONFIG, "plan label not in network"};
        if (bit >= 64) throw Failure{RCSG_ERR_CONFIG, "more than 64 fixed qubits"};
        roles[l].role = kVar;
        roles[l].var_bit = static_cast<int16_t>(bit++);
    }
    for (int b = 0; b < plan.n_sliced; ++b) {
        const int l = plan.sliced[b];
        if (l < 0 || l >= net.n_labels) throw Failure{RCSG_ERR_CONFIG, "plan label not in network"};
        roles[l].role = kPass;
        roles[l].src = PassSrc{1, 0, static_cast<int16_t>(b)};
    }
    for (int b = 0; b < plan.n_broken; ++b) {
        const int l = plan.broken[b];
        if (l < 0 || l >= net.n_labels) throw Failure{RCSG_ERR_CONFIG, "plan label not in network"};
        roles[l].role = kPass;
        roles[l].src = PassSrc{2, 0, static_cast<int16_t>(b)};
    }
    return roles;
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return record_error(RCSG_OK, "", -1);
    } catch (const Failure& e) {
        return record_error(e.code, e.msg, e.step);
    } catch (const std::bad_alloc&) {
        return record_error(RCSG_ERR_CAPACITY, "host allocation failed", -1);
    } catch (const std::exception& e) {
        return record_error(RCSG_ERR_DEVICE, e.what(), -1);
    }
}

}  // namespace

struct rcsg_context {
    std::vector<int> devices;
    std::vector<ncclComm_t> comms;
    std::vector<cudaStream_t> streams;
    ~rcsg_context() {
        for (size_t i = 0; i < devices.size(); ++i) {
            cudaSetDevice(devices[i]);
            if (i < comms.size() && comms[i] && nccl().CommDestroy) nccl().CommDestroy(comms[i]);
            if (i < streams.size() && streams[i]) cudaStreamDestroy(streams[i]);
        }
    }
};

struct rcsg_multi {
    rcsg_context* ctx = nullptr;
    std::vector<std::unique_ptr<Program>> progs;  // one per context device
    int n_sliced = 0, n_broken = 0;
    int n_blocks = 8;
};

extern "C" {

int rcsg_init(const int32_t* devices, int32_t n_devices, rcsg_context** out) {
    return guard([&] {
        if (!devices || n_devices < 1 || !out) throw Failure{RCSG_ERR_CONFIG, "rcsg_init needs >= 1 device"};
        int count = 0;
        CUDA_OK(cudaGetDeviceCount(&count));
        auto ctx = std::make_unique<rcsg_context>();
        for (int i = 0; i < n_devices; ++i) {
            if (devices[i] < 0 || devices[i] >= count)
                throw Failure{RCSG_ERR_CONFIG, "device " + std::to_string(devices[i]) + " not present"};
            if (std::find(ctx->devices.begin(), ctx->devices.end(), devices[i]) != ctx->devices.end())
                throw Failure{RCSG_ERR_CONFIG, "device listed twice"};
            ctx->devices.push_back(devices[i]);
        }
        ctx->streams.assign(n_devices, nullptr);
        for (int i = 0; i < n_devices; ++i) {
            CUDA_OK(cudaSetDevice(devices[i]));
            CUDA_OK(cudaStreamCreateWithFlags(&ctx->streams[i], cudaStreamNonBlocking));
        }
        if (n_devices > 1) {
            if (!nccl().CommInitAll) throw Failure{RCSG_ERR_DEVICE, "NCCL (libnccl.so.2) not available"};
            ctx->comms.assign(n_devices, nullptr);
            nccl_ok(nccl().CommInitAll(ctx->comms.data(), n_devices, ctx->devices.data()), "ncclCommInitAll");
        }
        CUDA_OK(cudaSetDevice(devices[0]));
        *out = ctx.release();
    });
}

int rcsg_context_free(rcsg_context* ctx) {
    return guard([&] { delete ctx; });
}

int rcsg_context_devices(rcsg_context* ctx, int32_t* n) {
    return guard([&] {
        if (!ctx || !n) throw Failure{RCSG_ERR_CONFIG, "null argument"};
        *n = static_cast<int32_t>(ctx->devices.size());
    });
}

int rcsg_context_compile(rcsg_context* ctx, const rcsg_network_desc* net, const rcsg_plan_desc* plan,
                         int32_t precision, uint64_t mem_budget_bytes, int32_t n_blocks, rcsg_multi** out) {
    return guard([&] {
        if (!ctx || !net || !plan || !out) throw Failure{RCSG_ERR_CONFIG, "null argument"};
        auto m = std::make_unique<rcsg_multi>();
        m->ctx = ctx;
        m->n_sliced = plan->n_sliced;
        m->n_broken = plan->n_broken;
        m->n_blocks = n_blocks > 0 ? n_blocks : 8;
        const std::vector<LabelRole> roles = roles_for_groups(*net, *plan);
        for (int dev : ctx->devices) {
            CUDA_OK(cudaSetDevice(dev));
            m->progs.push_back(std::make_unique<Program>(*net, *plan, roles, precision, mem_budget_bytes));
        }
        CUDA_OK(cudaSetDevice(ctx->devices[0]));
        *out = m.release();
    });
}

int rcsg_multi_free(rcsg_multi* m) {
    return guard([&] {
        if (!m) return;
        for (size_t i = 0; i < m->progs.size(); ++i) {
            cudaSetDevice(m->ctx->devices[i]);
            m->progs[i].reset();
        }
        cudaSetDevice(m->ctx->devices[0]);
        delete m;
    });
}

int rcsg_multi_contract_groups(rcsg_multi* m, uint64_t n_groups, const uint64_t* group_fixed, uint64_t n_configs,
                               const uint64_t* configs, uint64_t slice_begin, uint64_t slice_end, int32_t n_used,
                               double* out_amps, rcsg_stats* stats) {
    return guard([&] {
        if (!m || !group_fixed || !out_amps) throw Failure{RCSG_ERR_CONFIG, "null argument"};
        if (n_groups < 1) throw Failure{RCSG_ERR_CONFIG, "group count must be >= 1"};
        if (n_configs == 0 && m->n_broken > 0)
            throw Failure{RCSG_ERR_CONFIG, "plan has broken edges; exact contraction needs a plan without them"};
        if (n_configs > 0 && m->n_broken == 0) throw Failure{RCSG_ERR_CONFIG, "broken-edge labels do not match the plan"};
        if (slice_end > (uint64_t{1} << m->n_sliced) || slice_begin >= slice_end)
            throw Failure{RCSG_ERR_CONFIG, "slice range outside [0, 2^|sliced|)"};
        rcsg_context* ctx = m->ctx;
        const int nd = std::max(1, std::min<int>(n_used > 0 ? n_used : static_cast<int>(ctx->devices.size()),
                                                 static_cast<int>(ctx->devices.size())));
        // canonical blocks of the slice range (independent of nd)
        const uint64_t span = slice_end - slice_begin;
        const int nb = static_cast<int>(std::min<uint64_t>(static_cast<uint64_t>(m->n_blocks), span));
        std::vector<std::pair<uint64_t, uint64_t>> blocks(nb);
        for (int b = 0; b < nb; ++b)
            blocks[b] = {slice_begin + span * b / nb, slice_begin + span * (b + 1) / nb};
        const int64_t per = static_cast<int64_t>(n_groups) << m->progs[0]->out_rank();
        const int64_t n_el = per * 2;  // interleaved doubles per partial
        const std::vector<uint64_t> groups(group_fixed, group_fixed + n_groups);
        const std::vector<uint64_t> cfgs(configs, configs + n_configs);
        // device 0 holds every block's partial (the gather target); others hold their own
        std::vector<double*> part(nd, nullptr);
        std::vector<std::vector<int>> mine(nd);
        for (int b = 0; b < nb; ++b) mine[b % nd].push_back(b);
        std::vector<Failure> errs(nd, Failure{RCSG_OK, "", -1});
        std::vector<rcsg_stats> st(nd);
        auto run_device = [&](int d) {
            try {
                CUDA_OK(cudaSetDevice(ctx->devices[d]));
                const size_t slots = d == 0 ? static_cast<size_t>(nb) : mine[d].size();
                CUDA_OK(cudaMalloc(&part[d], std::max<size_t>(slots, 1) * n_el * sizeof(double)));
                CUDA_OK(cudaMemsetAsync(part[d], 0, slots * n_el * sizeof(double), m->progs[d]->stream()));
                for (size_t j = 0; j < mine[d].size(); ++j) {
                    const int b = mine[d][j];
                    double* dst = part[d] + (d == 0 ? b : static_cast<int>(j)) * n_el;
                    m->progs[d]->run(groups, cfgs, blocks[b].first, blocks[b].second, dst, &st[d], true);
                }
            } catch (const Failure& f) {
                errs[d] = f;
            } catch (const std::exception& e) {
                errs[d] = Failure{RCSG_ERR_DEVICE, e.what(), -1};
            }
        };
        std::vector<std::thread> pool;
        for (int d = 1; d < nd; ++d) pool.emplace_back(run_device, d);
        run_device(0);
        for (auto& th : pool) th.join();
        auto free_parts = [&] {
            for (int d = 0; d < nd; ++d)
                if (part[d]) {
                    cudaSetDevice(ctx->devices[d]);
                    cudaFree(part[d]);
                }
            cudaSetDevice(ctx->devices[0]);
        };
        for (int d = 0; d < nd; ++d)
            if (errs[d].code != RCSG_OK) {
                free_parts();
                throw errs[d];
            }
        if (nd > 1) {  // gather the other devices' block partials into device 0's slots (one NCCL group)
            nccl_ok(nccl().GroupStart(), "ncclGroupStart");
            for (int d = 1; d < nd; ++d)
                for (size_t j = 0; j < mine[d].size(); ++j) {
                    const int b = mine[d][j];
                    nccl_ok(nccl().Send(part[d] + j * n_el, static_cast<size_t>(n_el), ncclFloat64, 0, ctx->comms[d],
                                        ctx->streams[d]),
                            "ncclSend");
                    nccl_ok(nccl().Recv(part[0] + b * n_el, static_cast<size_t>(n_el), ncclFloat64, d, ctx->comms[0],
                                        ctx->streams[0]),
                            "ncclRecv");
                }
            nccl_ok(nccl().GroupEnd(), "ncclGroupEnd");
            for (int d = 0; d < nd; ++d) {
                CUDA_OK(cudaSetDevice(ctx->devices[d]));
                CUDA_OK(cudaStreamSynchronize(ctx->streams[d]));
            }
        }
        CUDA_OK(cudaSetDevice(ctx->devices[0]));
        double* sum = nullptr;
        CUDA_OK(cudaMalloc(&sum, n_el * sizeof(double)));
        const int grid = static_cast<int>(std::min<int64_t>((n_el + 255) / 256, 148 * 8));
        block_sum_kernel<<<grid, 256, 0, ctx->streams[0]>>>(part[0], nb, n_el, sum);
        CUDA_OK(cudaGetLastError());
        CUDA_OK(cudaMemcpyAsync(out_amps, sum, n_el * sizeof(double), cudaMemcpyDeviceToHost, ctx->streams[0]));
        CUDA_OK(cudaStreamSynchronize(ctx->streams[0]));
        cudaFree(sum);
        free_parts();
        if (stats) {
            *stats = rcsg_stats{};
            for (int d = 0; d < nd; ++d) {
                stats->plan_flops += st[d].plan_flops;
                stats->executed_flops += st[d].executed_flops;
                stats->arena_bytes = std::max(stats->arena_bytes, st[d].arena_bytes);
                stats->kernel_launches += st[d].kernel_launches;
                stats->passes += st[d].passes;
                stats->device_ms = std::max(stats->device_ms, st[d].device_ms);
            }
        }
    });
}

}  // extern "C"
