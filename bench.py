#!/usr/bin/env python3
"""Benchmark of the B200 sliced-contraction sampler (BASELINE.json metric).

Workload (BASELINE configs[1], "cfg2"): grid(5,6) 30-qubit random circuit,
14 cycles, seed 1, l = 6 open qubits {0..5}, the reference planner's plan with
exactly 2^8 slices (budget 3*2^30 B, effort low), K = 0, a batch of M candidate
groups drawn with the harness stream Rng(seed).split(0xca11d).  One STEP = one
slice contraction: slice s of the plan executed for all M groups on one GPU
(accumulated into the group amplitudes).  Multi-GPU: each rank contracts its
own slices (s = rank, rank+N, ...) with no data-path collective; one NCCL
all-reduce of the [M][2^l] partial amplitudes closes the timed region (the
slice sum is the path's only exchange step).  Weak scaling.

Metric: slice contractions/s (whole job).  Also reported: group-slice pairs/s,
complex TFLOP/s (executed and reference-equivalent, 8 real FLOP per complex
MAC), the tcgen05 GEMM roofline, a CPU baseline (the reference library on the
host cores), an end-to-end number through the public API with host buffers,
and XEB / samples/s of the cfg1 sampler pipeline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--groups M] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG2 = dict(n=30, cycles=14, topology="grid(5,6)", seed=1, open=list(range(6)), budget=3 << 30,
            effort="low")
WORKLOAD = "cfg2: grid(5,6) n=30 cycles=14 seed=1 l=6 open={0..5}, 2^8 slices (budget 3*2^30 B), K=0"
METRIC = "slice contractions/s"
DTYPES = {"f16": "f16 storage (per-tensor 2^e scales), tcgen05 kind::f16, f32 accumulate",
          "tf32": "f32 storage, tcgen05 kind::tf32, f32 accumulate",
          "bf16": "bf16 storage, tcgen05 kind::f16 (bf16), f32 accumulate",
          "f32": "f32 (SIMT)", "f64": "f64 (SIMT)"}
UNIT = "slice-contractions/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=256)  # all 2^8 slices of cfg2
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--groups", type=int, default=1024)  # cfg2 smoke scale M = 2^10
    ap.add_argument("--precision", default="f16", choices=["f16", "tf32", "bf16", "f32", "f64"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-xeb", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class Clocks:
    """nvidia-smi clock / throttle sampling during the timed region."""

    def __init__(self, index: int):
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{index}.csv")
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "40"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return None
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


_REF_PROBLEM = []


def cpu_reference_sample(threads: int, n_pairs: int | None = None, first: int = 0):
    """The reference executor (oracle/_ref, unmodified reference sources) on the
    host cores: execute_assignment on `n_pairs` (default `threads`) distinct
    (group, slice) pairs, spread over `threads` threads, of the same circuit
    planned with a tighter budget (2^27 B -> 15 sliced labels, ~1e10 FLOP per
    pair) so one pair takes seconds; returns measured FLOP/s."""
    from oracle import ref  # CPU baseline leg only
    if not _REF_PROBLEM:
        _REF_PROBLEM.append(ref.RefProblem(CFG2["n"], CFG2["cycles"], CFG2["topology"], CFG2["seed"],
                                           CFG2["open"], 1 << 27, "low").build())
    p = _REF_PROBLEM[0]
    fixed = ref.candidates(30, CFG2["open"], 1, ref.split_next(1, 0xCA11D))[0][0]
    n_pairs = n_pairs or threads
    slices = [(first + i) % (1 << len(p.plan["sliced"])) for i in range(n_pairs)]
    _, secs = p.slices_mt(int(fixed), slices, threads)
    flops = n_pairs * p.plan["flops_per_slice"]
    return flops / secs, secs, p.plan["flops_per_slice"], len(p.plan["sliced"])


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    import paper_2406_18889_b200 as pb  # host planner only (same plan as the reference's)
    threads = os.cpu_count() or 1
    p = pb.Problem(CFG2["n"], CFG2["cycles"], CFG2["topology"], CFG2["seed"], CFG2["open"], CFG2["budget"],
                   CFG2["effort"]).build()
    fps = p.plan["flops_per_slice"]
    # one step = one (group, slice) pair of the reference executor; the W warm-up
    # pairs and then the timed pairs each run spread over all host threads
    cpu_reference_sample(threads, max(args.warmup, 1), 0)
    # at least one pair per host thread (whole waves), so a small K still uses every core
    n_pairs = -(-max(args.steps, threads) // threads) * threads
    rate, secs, f_sample, _ = cpu_reference_sample(threads, n_pairs, args.warmup)
    pairs_per_s = rate / fps
    value = pairs_per_s / args.groups
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / value, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128 (f64)", "data": "synthetic",
            "config": {"workload": WORKLOAD, "groups_per_slice": args.groups},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": f"reference execute_assignment on {n_pairs} (group, slice) pairs over "
                                       f"{threads} threads in {secs:.1f} s, same circuit planned at budget 2^27 B "
                                       f"({f_sample:.3e} FLOP/pair); measured {rate / 1e9:.2f} GFLOP/s "
                                       f"extrapolated to the bench plan ({fps:.3e} FLOP/pair) x {args.groups} groups"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def xeb_cfg1(pb, precision):
    """cfg1 sampler pipeline on the GPU: grid(3,4) 12q 8 cycles, l=3, M=512,
    K=2 broken edges (m=1) -> amplitudes -> top-k (k=64) / direct sampling ->
    XEB against exact probabilities from the exact (K=0) f64 contraction of the
    same groups."""
    import numpy as np
    import torch
    n, l, M, k = 12, 3, 512, 64
    t0 = time.perf_counter()
    approx = pb.Problem(n, 8, "grid(3,4)", 1, list(range(l)), 1 << 30, "low", 2, 1).build()
    exact = pb.Problem(n, 8, "grid(3,4)", 1, list(range(l)), 1 << 30, "low").build()
    fixed, _ = pb.build_candidate_set(n, list(range(l)), M, pb.split_next(1, 0xCA11D))
    acc = torch.zeros(M * (1 << l) * 2, dtype=torch.float64, device="cuda")
    approx.contract_groups_device(fixed, acc.data_ptr(), precision="f64")
    top = pb.api.top_k_from_device_amps(n, list(range(l)), fixed, acc.data_ptr(), k)
    direct = pb.api.direct_from_device_amps(n, list(range(l)), fixed, acc.data_ptr(), pb.split_next(1, 0xD1EC7))
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    ex = exact.contract_groups(fixed, precision="f64", configs=None)
    ap = acc.cpu().numpy().view(np.complex128).reshape(M, -1)
    q = {}
    for g, fb in enumerate(fixed):
        for i in range(1 << l):
            q[pb.member(n, list(range(l)), int(fb), i)] = abs(ex[g, i]) ** 2
    xeb_top = pb.xeb(n, [q[int(s)] for s in top])
    xeb_dir = pb.xeb(n, [q[int(s)] for s in direct])
    fid = abs(np.vdot(ex.reshape(-1), ap.reshape(-1))) ** 2 / (np.vdot(ap, ap).real * np.vdot(ex, ex).real)
    return {"config": "cfg1 grid(3,4) n=12 cycles=8 l=3 M=512 K=2 m=1",
            "xeb_topk": xeb_top, "k": k, "predicted_topk": fid * np.log(M * (1 << l) / k),
            "xeb_direct": xeb_dir, "fidelity_over_candidates": fid,
            "samples_per_s": (k + M) / (t1 - t0)}


def xeb_cfg2(pb, p, fixed, precision):
    """cfg2 end to end at n = 30 against the exact GPU statevector (SURVEY §8f
    row 3): all 2^8 slices for the M groups (K = 0, so the amplitudes are the
    exact ones up to the storage precision) -> top-k with k = M (the paper's k =
    #groups) and one direct sample per group -> linear XEB from the ideal
    probabilities; plus the amplitude fidelity of all M * 2^l candidates."""
    import numpy as np
    import torch
    n, l, M = 30, 6, len(fixed)
    P = 1 << l
    acc = torch.zeros(M * P * 2, dtype=torch.float64, device="cuda")
    t0 = time.perf_counter()
    for s0 in range(0, p.n_slices, 8):
        p.contract_groups_device(fixed, acc.data_ptr(), precision=precision, configs=None, slices=(s0, s0 + 8),
                                 sync=False)
    p.sync(precision)
    top = pb.api.top_k_from_device_amps(n, CFG2["open"], fixed, acc.data_ptr(), M)
    direct = pb.api.direct_from_device_amps(n, CFG2["open"], fixed, acc.data_ptr(), pb.split_next(1, 0xD1EC7))
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    state = torch.empty(1 << n, dtype=torch.complex128, device="cuda")
    p.exact_state_device(state.data_ptr())
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    probs = (state.real ** 2 + state.imag ** 2)
    q_top = probs[torch.as_tensor(top.astype(np.int64), device="cuda")].cpu().numpy()
    q_dir = probs[torch.as_tensor(direct.astype(np.int64), device="cuda")].cpu().numpy()
    cand = np.array([pb.member(n, CFG2["open"], int(f), i) for f in fixed for i in range(P)], np.int64)
    ex = state[torch.as_tensor(cand, device="cuda")].cpu().numpy()
    del state, probs
    ap = acc.cpu().numpy().view(np.complex128).reshape(-1)
    fid = abs(np.vdot(ex, ap)) ** 2 / (np.vdot(ap, ap).real * np.vdot(ex, ex).real)
    return {"config": f"cfg2 grid(5,6) n=30 cycles=14 l=6 M={M} K=0, all 256 slices, {precision}",
            # Porter-Thomas: keeping the top fraction k / (M 2^l) of exact probabilities gives XEB = ln(M 2^l / k)
            "xeb_topk": pb.xeb(n, q_top), "k": M, "predicted_topk_exact": float(np.log(M * P / M)),
            "xeb_direct": pb.xeb(n, q_dir), "amplitude_fidelity_vs_exact": float(fid),
            "contract_and_sample_s": t1 - t0, "statevector_s": t2 - t1,
            "note": "ideal probabilities from the GPU statevector (simulate_exact, bit-exact with the reference)"}


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2406_18889_b200 as pb
    from paper_2406_18889_b200._native import rcsg_stats

    torch.cuda.set_device(local)
    pb.api.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    hbm_peak, bf16_peak, peak_kind = peaks()

    p = pb.Problem(CFG2["n"], CFG2["cycles"], CFG2["topology"], CFG2["seed"], CFG2["open"], CFG2["budget"],
                   CFG2["effort"]).build()
    assert p.n_slices == 256, p.n_slices
    M = args.groups
    fixed, dups = pb.build_candidate_set(30, CFG2["open"], M, pb.split_next(1, 0xCA11D))
    P = 1 << p.n_open
    acc = torch.zeros(M * P * 2, dtype=torch.float64, device="cuda")
    stream = torch.cuda.ExternalStream(p.stream(args.precision))

    # a step is one slice contraction; one call contracts an aligned block of S
    # consecutive slices (one device pass per slice, or per slice batch when the
    # executor batches clean low sliced labels)
    S = min(8, p.n_slices)
    n_calls = (args.steps + S - 1) // S

    def block_of(i):
        return (rank + i * world) % (p.n_slices // S)

    def step(i, st=None, sync=True, count=None):
        s = block_of(i) * S
        return p.contract_groups_device(fixed, acc.data_ptr(), precision=args.precision, configs=None,
                                        slices=(s, s + (count or S)), stats=st, sync=sync)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # L2 flush between timed steps: a 256 MiB write (> 126 MB L2) on the program's
    # stream, outside each step's event pair
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(n_calls)]
    clocks = Clocks(local)
    st = rcsg_stats()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with torch.cuda.stream(stream):
        for i in range(n_calls):
            flush.fill_(i & 0xFF)
            evs[i][0].record(stream)
            count = min(S, args.steps - i * S)
            step(args.warmup + i, st, sync=False, count=count)  # enqueue only; checked by p.sync below
            if i == n_calls - 1 and world > 1:
                dist.all_reduce(acc)  # the slice sum across ranks
            evs[i][1].record(stream)
    p.sync(args.precision)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = sum(a.elapsed_time(b) for a, b in evs)
    clk = clocks.stop()
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * args.steps / (ms_max / 1e3)
    exec_flops = st.executed_flops
    plan_flops = st.plan_flops

    # kernel-class breakdown from one profiled step (outside the timed region)
    p.set_profile(True)
    pst = rcsg_stats()
    step(args.warmup + args.steps, pst)
    p.set_profile(False)
    tc_tflops = pst.gemm_tc_flops / (pst.gemm_tc_ms * 1e-3) / 1e12 if pst.gemm_tc_ms else 0.0
    # dense tensor peak of the MMA kind the precision uses: fp16/bf16 = measured bf16; tf32 = half of it
    tc_peak = bf16_peak / 2.0 if args.precision == "tf32" else bf16_peak
    peak_note = (f"tf32 dense = 1/2 of {peak_kind} bf16 {bf16_peak:.1f} TF/s" if args.precision == "tf32"
                 else f"{peak_kind} dense bf16/fp16 peak {bf16_peak:.1f} TF/s")

    # roofline of the dominant kernel: the plan step with the longest launch of the profiled pass,
    # bound by its arithmetic intensity (algorithmic FLOPs / algorithmic bytes)
    classes = {0: "SIMT GEMM", 1: "tcgen05 GEMM (gemm_tc_persistent / gemm_tc_kernel)", 2: "permute", 3: "GEMV"}
    # average launch of the dominant plan step over the profiled pass (S launches), not its slowest
    top_ms = pst.top_ms_sum / pst.top_launches if pst.top_launches else pst.top_ms
    top_s = top_ms * 1e-3
    ai = pst.top_flops / pst.top_bytes if pst.top_bytes else float("inf")
    ridge = tc_peak * 1e12 / (hbm_peak * 1e9)
    if ai >= ridge:
        bound, ach, peak, unit = "tensor", pst.top_flops / top_s / 1e12, tc_peak, "TFLOP/s"
        pnote = peak_note
        algo = pst.top_flops
    else:
        bound, ach, peak, unit = "hbm", pst.top_bytes / top_s / 1e9, hbm_peak, "GB/s"
        pnote = f"{peak_kind} HBM copy bandwidth {hbm_peak:.1f} GB/s"
        algo = pst.top_bytes
    traffic = None
    try:  # dram read + write of this launch from the committed ncu --set full capture
        with open(os.path.join(ROOT, "profiles", "top_kernel_traffic.json")) as f:
            tk = json.load(f)
        if int(tk.get("plan_step", -1)) == int(pst.top_step) and tk.get("precision") == args.precision:
            traffic = int(tk["dram_bytes"])
    except Exception:
        pass
    roofline = {"bound": bound, "kernel": f"plan step {pst.top_step}: {classes.get(int(pst.top_class), '?')}",
                "achieved": ach, "peak": peak, "unit": unit, "frac": ach / peak, "traffic": traffic,
                "algorithmic_per_launch": algo, "launch_ms": top_ms, "launches_averaged": int(pst.top_launches),
                "slowest_launch_ms": pst.top_ms, "flops": pst.top_flops,
                "bytes": pst.top_bytes, "intensity_flop_per_byte": ai, "ridge_flop_per_byte": ridge,
                "peak_note": pnote,
                "share_of_step": pst.top_ms_sum / pst.device_ms if pst.device_ms and pst.top_launches
                else (pst.top_ms * S / pst.device_ms if pst.device_ms else None),  # profiled call = S passes
                "all_tensor_core_launches": {"achieved_tflops": tc_tflops, "frac_of_tensor_peak": tc_tflops / tc_peak,
                                             "share_of_step": pst.gemm_tc_ms / pst.device_ms if pst.device_ms else None}}

    # end-to-end through the public API with host buffers (rank 0 work pattern on each rank)
    e2e = None
    if not args.no_e2e:
        K = max(2, min(n_calls, 8))  # calls of S slices each
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(K):
            s = block_of(i) * S
            out = p.contract_groups(fixed, precision=args.precision, configs=None, slices=(s, s + S))
        t1 = time.perf_counter()
        e2e = {"value": world * K * S / (t1 - t0), "unit": UNIT,
               "h2d_bytes_per_step": int(fixed.nbytes) / S, "d2h_bytes_per_step": int(out.nbytes) / S,
               "api": f"Problem.contract_groups (host in/out), {S} slices per call"}
        if world > 1:
            tt = torch.tensor([t1 - t0], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e["value"] = world * K * S / float(tt.item())

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            rate, secs, f_sample, _ = cpu_reference_sample(os.cpu_count() or 1)
            cpu_val = rate / p.plan["flops_per_slice"] / M
            cpu = {"value": cpu_val, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"reference execute_assignment (oracle/_ref) on {os.cpu_count()} (group, slice) pairs "
                             f"in parallel, cfg2 circuit planned at 2^27 B ({f_sample:.3e} FLOP/pair), {secs:.1f} s; "
                             f"{rate / 1e9:.2f} GFLOP/s extrapolated to {p.plan['flops_per_slice']:.3e} FLOP/pair "
                             f"x {M} groups"}
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    xeb = None
    if rank == 0 and not args.no_xeb:
        try:
            xeb = xeb_cfg1(pb, args.precision)
        except Exception as e:  # pragma: no cover
            xeb = {"error": str(e)}
        if world == 1:
            try:
                xeb = {"cfg1": xeb, "cfg2": xeb_cfg2(pb, p, fixed, args.precision)}
            except Exception as e:  # pragma: no cover
                xeb = {"cfg1": xeb, "cfg2": {"error": str(e)}}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": DTYPES[args.precision],
            "data": "synthetic (random circuit of the named shape)",
            "config": {"workload": WORKLOAD, "groups_per_slice": M, "duplicate_groups": int(dups),
                       "slices_per_call": S,
                       "precision": args.precision, "l2": "flushed between timed steps (256 MiB write, "
                       f"outside the per-step events); arena {st.arena_bytes / 2**30:.2f} GiB per GPU",
                       "parallelism": f"slice-sharded x{world}"},
            "group_slice_pairs_per_s": value * M,
            "complex_tflops_executed": exec_flops * world / (ms_max * 1e-3) / 1e12,
            "complex_tflops_reference_equivalent": plan_flops * world / (ms_max * 1e-3) / 1e12,
            "gpu_launches": int(st.kernel_launches),
            "roofline": roofline,
            "kernel_breakdown_ms": {"per": f"one profiled pass of {S} slices (serialised launches)",
                                    "step": pst.device_ms, "gemm_tc": pst.gemm_tc_ms,
                                    "gemm_other": pst.gemm_ms - pst.gemm_tc_ms, "permute": pst.permute_ms,
                                    "permute_gbs": pst.permute_bytes / (pst.permute_ms * 1e-3) / 1e9
                                    if pst.permute_ms else None, "hbm_peak_gbs": hbm_peak},
            "e2e": e2e, "cpu_baseline": cpu, "xeb": xeb, "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
