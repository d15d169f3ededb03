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

Metric: slice contractions/s (whole job).  The headline line is the north
star's primary precision, tf32 (fp32 storage, tcgen05 kind::tf32 - the paper's
tensor-core precision); the fp16 mode is measured in the same run
under "f16".  Also reported: group-slice pairs/s, complex TFLOP/s (executed and
reference-equivalent, 8 real FLOP per complex MAC), the roofline of the dominant
kernel per mode, a CPU baseline (the reference library on the host cores, same
plan), end-to-end numbers through the public API with host buffers (warm, and
cold: a fresh program and candidate set, binding inside the timed region), the
fused post-processing kernel's HBM GB/s at M = 2^20, and XEB.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--groups M] [--impl reference]
"""
from __future__ import annotations

import argparse
import datetime as _dt
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
          "3xtf32": "f32 storage, split hi + lo operands on tcgen05 kind::tf32 (3 products), f32 accumulate",
          "bf16": "bf16 storage, tcgen05 kind::f16 (bf16), f32 accumulate",
          "f32": "f32 (SIMT)", "f64": "f64 (SIMT)"}
UNIT = "slice-contractions/s"


def config_of(groups: int) -> dict:
    """The workload description; identical in both arms (the driver compares it)."""
    return {"workload": WORKLOAD, "groups_per_slice": groups}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=256)  # all 2^8 slices of cfg2
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--groups", type=int, default=1024)  # cfg2 smoke scale M = 2^10
    ap.add_argument("--precision", default="tf32", choices=["f16", "tf32", "3xtf32", "bf16", "f32", "f64"])
    ap.add_argument("--alt-precision", default="f16", choices=["none", "f16", "tf32", "bf16"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-xeb", action="store_true")
    ap.add_argument("--no-post", action="store_true")
    ap.add_argument("--scale-configs", default="cfg3,cfg4,cfg5",
                    help="BASELINE configs 3-5 measured per slice with the scale planner (comma list, or none)")
    ap.add_argument("--cfg4-slices", type=int, default=1024, help="cfg4 fixed slice subset (BASELINE: 2^10)")
    ap.add_argument("--replan", action="store_true",
                    help="cfg3-5: run the scale planner in this process instead of importing plans/<cfg>.json")
    ap.add_argument("--ref-pairs", type=int, default=0,
                    help="(group, slice) pairs the reference executor runs (default: one per host core, >= 16)")
    ap.add_argument("--ref-budget", type=int, default=CFG2["budget"],
                    help="(tests only) plan budget of the reference sample; the default is the bench plan")
    return ap.parse_args()


# stdout carries exactly one JSON line: library banners (NCCL version, ...) that
# write to fd 1 are sent to stderr, the result line goes to the original stdout
_RESULT_FD = None


def emit(line: dict) -> None:
    data = (json.dumps(line) + "\n").encode()
    if _RESULT_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        os.write(_RESULT_FD, data)


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
    """nvidia-smi clock / throttle sampling; started before the warm-up so it is
    running when the timed region begins, and summarised over the samples whose
    timestamps fall inside [mark_begin, mark_end]."""

    def __init__(self, index: int):
        self.proc = None
        self.window = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{index}.csv")
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={index}",
                 "--query-gpu=timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=self.f, stderr=subprocess.DEVNULL)
            t0 = time.time()  # wait for the first sample (the sampler needs ~0.2-1 s to start)
            while time.time() - t0 < 5 and os.path.getsize(self.path) == 0:
                time.sleep(0.05)
        except Exception:
            self.proc = None

    def mark(self, begin: bool):
        now = time.time()
        if begin:
            self.window = [now, None]
        elif self.window:
            self.window[1] = now

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.1)
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        lo, hi = (self.window or [0, 1e30])
        hi = hi or 1e30
        sm, mx, reasons, n_all = [], 0.0, set(), 0
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                ts = _dt.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                clk, cmax = float(parts[1]), float(parts[2])
            except ValueError:
                continue
            n_all += 1
            if not (lo - 0.03 <= ts <= hi + 0.03):
                continue
            sm.append(clk)
            mx = max(mx, cmax)
            for name, val in zip(names, parts[4:8]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "samples_total": n_all}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "timed_region_s": hi - lo}


# ---- the reference's own CPU executor (oracle/_ref) -----------------------------
def reference_sample(n_pairs: int, threads: int, budget: int, groups: int):
    """The reference executor (oracle/_ref: the unmodified reference sources) on
    the host cores, on the bench's own plan (the reference planner at the bench
    budget): execute_assignment on `n_pairs` (group, slice) pairs - group 0 of the
    bench's candidate set with slices spread over the range - `threads` at a
    time.  Nothing of the product package is imported."""
    from oracle import ref  # CPU baseline / reference arm only
    r = ref.RefProblem(CFG2["n"], CFG2["cycles"], CFG2["topology"], CFG2["seed"], CFG2["open"], budget,
                       CFG2["effort"]).build()
    n_sl = 1 << len(r.plan["sliced"])
    fixed = ref.candidates(CFG2["n"], CFG2["open"], groups, ref.split_next(CFG2["seed"], 0xCA11D))[0]
    slices = [(i * n_sl) // n_pairs % n_sl for i in range(n_pairs)]
    _, secs = r.slices_mt(int(fixed[0]), slices, threads)
    return {"secs": secs, "pairs": n_pairs, "threads": threads, "flops_per_pair": r.plan["flops_per_slice"],
            "n_slices": n_sl, "plan": f"reference planner, budget {budget} B: {len(r.plan['sliced'])} sliced labels, "
                                      f"{len(r.plan['steps'])} steps"}


def reference_line_fields(smp, groups):
    pairs_per_s = smp["pairs"] / smp["secs"]
    value = pairs_per_s / groups  # one slice contraction = `groups` (group, slice) pairs of this plan
    sample = (f"reference execute_assignment (oracle/_ref) on {smp['pairs']} (group, slice) pairs of the bench plan "
              f"({smp['plan']}, {smp['flops_per_pair']:.3e} FLOP/pair), {smp['threads']} threads, "
              f"{smp['secs']:.1f} s -> {pairs_per_s:.4g} pairs/s "
              f"({pairs_per_s * smp['flops_per_pair'] / 1e9:.2f} GFLOP/s); one slice contraction = {groups} pairs, "
              f"so value = pairs/s / {groups}; the full cfg2 run (256 slices x {groups} groups) is extrapolated")
    return value, sample


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    n_pairs = args.ref_pairs or max(16, threads)
    smp = reference_sample(n_pairs, threads, args.ref_budget, args.groups)
    value, sample = reference_line_fields(smp, args.groups)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / value, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128 (f64, the reference executor)",
            "data": "synthetic", "config": config_of(args.groups),
            "timed_region_s": smp["secs"],
            "extrapolated": "one slice contraction of the CPU executor takes ms_per_step; the timed region is "
                            f"{smp['pairs']} (group, slice) pairs ({smp['secs']:.1f} s), not K whole steps",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)
    return 0


# ---- our arm ---------------------------------------------------------------------
def traffic_for(step: int, precision: str):
    """DRAM read + write of the dominant launch from a committed ncu --set full
    capture (profiles/top_kernel_traffic.json), if one matches this step."""
    try:
        with open(os.path.join(ROOT, "profiles", "top_kernel_traffic.json")) as f:
            tk = json.load(f)
    except Exception:
        return None
    for e in tk.get("entries", [tk]):
        if int(e.get("plan_step", -1)) == int(step) and e.get("precision") == precision:
            return int(e["dram_bytes"])
    return None


def measure(pb, p, fixed, precision, args, rank, world, clocks=None):
    """Times args.steps slice contractions of the M groups at `precision`; returns
    the value, the dominant-kernel roofline and a kernel breakdown."""
    import torch
    import torch.distributed as dist
    from paper_2406_18889_b200._native import rcsg_stats
    hbm_peak, bf16_peak, peak_kind = peaks()
    M, P = len(fixed), 1 << p.n_open
    acc = torch.zeros(M * P * 2, dtype=torch.float64, device="cuda")
    stream = torch.cuda.ExternalStream(p.stream(precision))
    S = min(8, p.n_slices)  # slices per call: an aligned block of consecutive slices
    n_calls = (args.steps + S - 1) // S

    def block_of(i):
        return (rank + i * world) % (p.n_slices // S)

    def step(i, st=None, sync=True, count=None):
        s = block_of(i) * S
        return p.contract_groups_device(fixed, acc.data_ptr(), precision=precision, configs=None,
                                        slices=(s, s + (count or S)), stats=st, sync=sync)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    # L2 flush between timed steps: a 256 MiB write (> 126 MB L2) on the program's
    # stream, outside each step's event pair
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n_calls)]
    st = rcsg_stats()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    if clocks:
        clocks.mark(True)
    with torch.cuda.stream(stream):
        for i in range(n_calls):
            flush.fill_(i & 0xFF)
            evs[i][0].record(stream)
            count = min(S, args.steps - i * S)
            step(args.warmup + i, st, sync=False, count=count)  # enqueue only; checked by p.sync below
            if i == n_calls - 1 and world > 1:
                dist.all_reduce(acc)  # the slice sum across ranks
            evs[i][1].record(stream)
    p.sync(precision)
    torch.cuda.synchronize()
    if clocks:
        clocks.mark(False)
    if world > 1:
        dist.barrier()
    ms = sum(a.elapsed_time(b) for a, b in evs)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * args.steps / (ms_max / 1e3)

    # kernel-class breakdown and the dominant launch from one profiled call (outside the timed region)
    p.set_profile(True)
    step(args.warmup + args.steps, rcsg_stats())  # first profiled call: per-launch event setup
    pst = rcsg_stats()
    step(args.warmup + args.steps + 1, pst)
    p.set_profile(False)
    tc_peak = bf16_peak / 2.0 if precision == "tf32" else (bf16_peak / 6.0 if precision == "3xtf32" else bf16_peak)
    peak_note = (f"dense tf32 = 1/2 of the {peak_kind} dense bf16 {bf16_peak:.1f} TF/s (B200 tf32:bf16 = 1:2)"
                 if precision == "tf32" else
                 (f"3xtf32: three tf32 products per real product, 1/6 of the {peak_kind} dense bf16 {bf16_peak:.1f}"
                  " TF/s" if precision == "3xtf32" else f"{peak_kind} dense bf16/fp16 peak {bf16_peak:.1f} TF/s"))
    tc_tflops = pst.gemm_tc_flops / (pst.gemm_tc_ms * 1e-3) / 1e12 if pst.gemm_tc_ms else 0.0
    classes = {0: "SIMT GEMM", 1: "tcgen05 GEMM (gemm_tc_persistent)", 2: "permute", 3: "GEMV"}
    top_ms = pst.top_ms_sum / pst.top_launches if pst.top_launches else pst.top_ms
    top_s = top_ms * 1e-3
    ai = pst.top_flops / pst.top_bytes if pst.top_bytes else float("inf")
    ridge = tc_peak * 1e12 / (hbm_peak * 1e9)
    if ai >= ridge:
        bound, ach, peak, unit, pnote, algo = "tensor", pst.top_flops / top_s / 1e12, tc_peak, "TFLOP/s", peak_note, \
            pst.top_flops
    else:
        bound, ach, peak, unit, algo = "hbm", pst.top_bytes / top_s / 1e9, hbm_peak, "GB/s", pst.top_bytes
        pnote = f"{peak_kind} HBM copy bandwidth {hbm_peak:.1f} GB/s"
    nominal = ({"tf32": 1100.0, "3xtf32": 1100.0 / 3}.get(precision, 2250.0)) if bound == "tensor" else 7700.0
    roofline = {"bound": bound, "kernel": f"plan step {pst.top_step}: {classes.get(int(pst.top_class), '?')}",
                "achieved": ach, "peak": peak, "unit": unit, "frac": ach / peak,
                "traffic": traffic_for(pst.top_step, precision),
                "algorithmic_per_launch": algo, "launch_ms": top_ms, "launches_averaged": int(pst.top_launches),
                "slowest_launch_ms": pst.top_ms, "flops": pst.top_flops, "bytes": pst.top_bytes,
                "intensity_flop_per_byte": ai, "ridge_flop_per_byte": ridge, "peak_note": pnote,
                # the measured bf16 figure is a cuBLAS burst at the power cap; tf32 at 1/2 of it can sit below
                # what a kernel reaches at its own clock, so the nominal dense peak (B200_PROFILING.md) is
                # reported beside it
                "nominal_peak": nominal,
                "frac_of_nominal": ach / nominal,
                "share_of_step": pst.top_ms_sum / pst.device_ms if pst.device_ms and pst.top_launches else None,
                "all_tensor_core_launches": {"achieved_tflops": tc_tflops, "frac_of_tensor_peak": tc_tflops / tc_peak,
                                             "share_of_step": pst.gemm_tc_ms / pst.device_ms
                                             if pst.device_ms else None}}
    return {"value": value, "ms_max": ms_max, "acc": acc, "S": S, "n_calls": n_calls, "block_of": block_of,
            "exec_flops": st.executed_flops, "plan_flops": st.plan_flops, "launches": int(st.kernel_launches),
            "arena": st.arena_bytes, "roofline": roofline,
            "breakdown": {"per": f"one profiled call of {S} slices (serialised launches)", "step": pst.device_ms,
                          "gemm_tc": pst.gemm_tc_ms, "gemm_other": pst.gemm_ms - pst.gemm_tc_ms,
                          "permute": pst.permute_ms, "hbm_peak_gbs": hbm_peak}}


def e2e_warm(p, fixed, precision, res, world):
    """Through the public API with host buffers: group prefixes in, amplitudes
    out, S slices per call, on the bound program."""
    import torch
    import torch.distributed as dist
    # a user call covers a block of S consecutive slices (one H2D of the group
    # prefixes, one D2H of the amplitudes per call); K calls cover every slice of
    # this rank once (the timed device run's work), after one untimed call
    S = min(32, p.n_slices)
    n_blocks = p.n_slices // S
    K = max(1, n_blocks // world)
    p.contract_groups(fixed, precision=precision, configs=None, slices=(0, S))
    torch.cuda.synchronize()
    calls = []
    for i in range(K):
        s = ((dist_env()[0] + i * world) % n_blocks) * S
        t0 = time.perf_counter()
        out = p.contract_groups(fixed, precision=precision, configs=None, slices=(s, s + S))
        calls.append(time.perf_counter() - t0)
    dt = sum(calls)
    if world > 1:
        tt = torch.tensor([dt], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
    return {"value": world * K * S / dt, "unit": UNIT, "h2d_bytes_per_step": int(fixed.nbytes) / S,
            "d2h_bytes_per_step": int(out.nbytes) / S,
            "api": f"Problem.contract_groups (host in/out), {K} calls of {S} slices (all slices of this rank), "
                   "program bound by an earlier call",
            "call_ms": [round(c * 1e3, 2) for c in calls]}


def e2e_cold(pb, precision, M, warm_value):
    """A fresh Problem (planning timed separately) and a NEW candidate set
    (Rng(2).split(0xca11d)); all 256 slices in one contract_groups call with host
    buffers, so compile, batch reassociation, fp16 calibration, binding, the
    phase-0/3 results, slice tables and graph capture are inside the timed call."""
    t0 = time.perf_counter()
    p2 = pb.Problem(CFG2["n"], CFG2["cycles"], CFG2["topology"], CFG2["seed"], CFG2["open"], CFG2["budget"],
                    CFG2["effort"]).build()
    t1 = time.perf_counter()
    fixed2, _ = pb.build_candidate_set(30, CFG2["open"], M, pb.split_next(2, 0xCA11D))
    out = p2.contract_groups(fixed2, precision=precision, configs=None)
    t2 = time.perf_counter()
    n = p2.n_slices
    return {"value": n / (t2 - t1), "unit": UNIT, "h2d_bytes_per_step": int(fixed2.nbytes) / n,
            "d2h_bytes_per_step": int(out.nbytes) / n, "slices": n, "contract_s": t2 - t1, "plan_s": t1 - t0,
            "bind_s_estimate": max(0.0, (t2 - t1) - n / warm_value) if warm_value else None,
            "api": "fresh Problem + new candidate set, one Problem.contract_groups call over all slices"}


SCALE_CFGS = {"cfg3": (53, 12, "sycamore53", "Sycamore-53 layout, m=12"),
              "cfg4": (53, 20, "sycamore53", "Sycamore-53 layout, m=20"),
              "cfg5": (60, 24, "zuchongzhi60", "Zuchongzhi-style 60 qubits, m=24")}


def scale_bench(pb, name, precision, n_slices, M=64, budget_log2=36, alt=None, alt_slices=64, trials=1024,
                compare=False, replan=False):
    """BASELINE configs 3-5 per slice: the scale planner (log-domain, batch-aware,
    stem-aware slicing; widest tensor 2^30 amplitudes incl. group variants at a
    2^36 B budget) plans the circuit for M = 64 groups; a fixed subset of the
    first `n_slices` slices runs timed (device events, after one warm-up call)
    and the full run is extrapolated from the per-slice time."""
    import torch
    from paper_2406_18889_b200._native import rcsg_stats
    hbm_peak, bf16_peak, peak_kind = peaks()
    n, m, topo, desc = SCALE_CFGS[name]
    plan_file = os.path.join(ROOT, "plans", f"{name}.json")
    t0 = time.perf_counter()
    if os.path.exists(plan_file) and not replan:
        # the committed plan file (plan.json; found offline by the same scale planner,
        # tools/plan_search.py): the measured plan is the same on every box
        meta = json.load(open(plan_file[:-5] + ".meta.json"))
        p = pb.Problem(n, m, topo, 1, CFG2["open"], 1 << budget_log2, "low").build(plan_json=open(plan_file).read())
        rep, source = meta["report"], f"plans/{name}.json (scale planner, {meta['trials']} trials, " \
                                      f"search seed {meta['seed']}; imported)"
    else:
        p = pb.Problem(n, m, topo, 1, CFG2["open"], 1 << budget_log2, "low").build(planner="scale", n_groups=M,
                                                                                   trials=trials)
        rep, source = p.plan_report or {}, f"scale planner, {trials} trials, planned in this run"
    plan_s = time.perf_counter() - t0
    fixed, _ = pb.build_candidate_set(n, CFG2["open"], M, pb.split_next(1, 0xCA11D))
    # device arena budget: 85% of the free HBM after torch returns its cache (the
    # executor's default is 70%; cfg5's tf32 arena is ~120 GB)
    torch.cuda.empty_cache()
    bud = int(torch.cuda.mem_get_info()[0] * 0.85)
    out = {"workload": f"{name}: {desc}, seed 1, l=6 open={{0..5}}, M={M} groups, K=0; "
                       f"scale planner, budget 2^{budget_log2} B",
           "plan": {"source": source, "sliced_labels": len(p.plan["sliced"]), "n_slices_log2": len(p.plan["sliced"]),
                    "flops_per_slice_per_group": p.plan["flops_per_slice"],
                    "log2_total_flops_batched": rep.get("log2_total_flops"),
                    "log2_flops_per_slice_batched": rep.get("log2_flops_per_slice_batched"),
                    "log2_widest_tensor": rep.get("log2_max_size"), "planner_s": rep.get("seconds"),
                    "build_s": plan_s}}
    for prec, ns in ((precision, n_slices), (alt, alt_slices)):
        if not prec:
            continue
        try:
            out[prec] = scale_mode(pb, p, fixed, prec, ns, M, bud, bf16_peak, peak_kind)
        except Exception as e:  # pragma: no cover - reported per mode
            out[prec] = {"error": str(e)}
        p.release()  # one mode's arena at a time (cfg5's is ~120 GB at tf32)
    if compare and alt and all("error" not in out.get(x, {"error": 1}) for x in (precision, alt)):
        # fp16-complex tensor-core mode against the fp32-storage (tf32) mode on the same two slices
        a = p.contract_groups(fixed, precision=precision, configs=None, slices=(0, 2), budget=bud)
        p.release()
        b = p.contract_groups(fixed, precision=alt, configs=None, slices=(0, 2), budget=bud)
        p.release()
        import numpy as np
        errs = np.linalg.norm(b - a, axis=1) / np.maximum(np.linalg.norm(a, axis=1), 1e-300)
        out[f"{alt}_vs_{precision}"] = {
            "slices": [0, 2], "groups": M, "max_norm_rel": float(errs.max()),
            "median_norm_rel": float(np.median(errs)), "tolerance": 1e-2,
            "within_tolerance": bool(errs.max() <= 1e-2),
            "note": "both modes round every stored intermediate to an 11-bit significand (fp16 storage; tf32 "
                    "operands); over ~2000 steps each drifts ~1-2% from the fp32 SIMT result "
                    "(tools/precision_probe.py, profiles/r02/precision_probe.log), so the cfg2 tolerance "
                    "of 1e-2 does not hold between them at this depth"}
    return out


def scale_mode(pb, p, fixed, prec, ns, M, bud, bf16_peak, peak_kind):
    """One precision mode of scale_bench: warm-up slice, `ns` timed slices in
    calls of 8 (device events on the program's stream), one profiled slice."""
    import torch
    from paper_2406_18889_b200._native import rcsg_stats
    acc = torch.zeros(M * 64 * 2, dtype=torch.float64, device="cuda")
    stream = torch.cuda.ExternalStream(p.stream(prec, bud))
    S = 8
    t1 = time.perf_counter()
    p.contract_groups_device(fixed, acc.data_ptr(), precision=prec, configs=None, slices=(0, 1),
                             budget=bud)  # warm-up
    torch.cuda.synchronize()
    warm_s = time.perf_counter() - t1
    st = rcsg_stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for s0 in range(0, ns, S):
            p.contract_groups_device(fixed, acc.data_ptr(), precision=prec, configs=None,
                                     slices=(s0, min(s0 + S, ns)), budget=bud, stats=st, sync=False)
        e1.record(stream)
    p.sync(prec, bud)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    # two profiled slices, the second one reported (the first sets up the per-launch events)
    p.set_profile(True)
    p.contract_groups_device(fixed, acc.data_ptr(), precision=prec, configs=None, slices=(0, 1), budget=bud,
                             stats=rcsg_stats())
    pst = rcsg_stats()
    p.contract_groups_device(fixed, acc.data_ptr(), precision=prec, configs=None, slices=(1, 2), budget=bud,
                             stats=pst)
    p.set_profile(False)
    tc_peak = bf16_peak / 2.0 if prec == "tf32" else bf16_peak
    hbm_peak = peaks()[0]
    rate = ns / (ms / 1e3)
    exec_tf = st.executed_flops / (ms / 1e3) / 1e12
    top_s = pst.top_ms_sum / pst.top_launches * 1e-3 if pst.top_launches else pst.top_ms * 1e-3
    ai = pst.top_flops / pst.top_bytes if pst.top_bytes else float("inf")
    if ai >= tc_peak * 1e12 / (hbm_peak * 1e9):
        bound, ach, peak, unit = "tensor", pst.top_flops / top_s / 1e12 if top_s else None, tc_peak, "TFLOP/s"
    else:
        bound, ach, peak, unit = "hbm", pst.top_bytes / top_s / 1e9 if top_s else None, hbm_peak, "GB/s"
    res = {
        "value": rate, "unit": UNIT, "timed_slices": ns, "ms": ms, "warm_s": warm_s,
        "executed_tflops": exec_tf, "frac_of_dense_peak": exec_tf / tc_peak,
        "peak_tflops": tc_peak, "peak_note": ("dense tf32 = 1/2 of " if prec == "tf32" else "") +
        f"{peak_kind} dense bf16 {bf16_peak:.1f} TF/s",
        "roofline": {"bound": bound, "kernel": f"plan step {pst.top_step}: tcgen05 GEMM",
                     "achieved": ach, "peak": peak, "unit": unit, "frac": ach / peak if ach else None,
                     "flops": pst.top_flops, "bytes": pst.top_bytes, "launch_ms": top_s * 1e3,
                     "share_of_slice": pst.top_ms_sum / pst.device_ms if pst.device_ms else None,
                     "traffic": None},
        "tensor_core_share_of_slice": pst.gemm_tc_ms / pst.device_ms if pst.device_ms else None,
        "full_run_extrapolated_s_1gpu": p.n_slices / rate,
        "arena_gib": st.arena_bytes / 2 ** 30, "amps_finite": bool(torch.isfinite(acc).all().item())}
    del acc
    return res


def post_bench(pb, hbm_peak):
    """Fused post-processing kernel (rcsg_postprocess) at M = 2^20 groups, l = 6
    (64 Mi candidates, 1 GiB of f64 amplitudes resident in HBM): top-k with
    k = 2^20 (= M, the paper's k) and k = 2^15, direct sampling alone, and
    both fused into the same streaming pass.  GB/s = algorithmic bytes (amplitudes read once +
    samples written) / device time of the call."""
    import numpy as np
    import torch
    M, l, n = 1 << 20, 6, 30
    g = torch.Generator(device="cuda").manual_seed(1)
    amps = torch.randn((M << l) * 2, dtype=torch.float64, device="cuda", generator=g) * 2.0 ** -15
    fixed = np.random.default_rng(1).integers(0, 1 << (n - l), size=M, dtype=np.uint64)
    out = {}
    for name, k, direct in (("topk_k2^20", 1 << 20, None), ("topk_k2^15", 1 << 15, None), ("direct", 0, 7),
                            ("topk_k2^20+direct", 1 << 20, 7)):
        pb.api.postprocess_device_amps(n, CFG2["open"], fixed, amps.data_ptr(), k, direct_seed=direct)
        best = None
        for _ in range(5):
            _, _, st = pb.api.postprocess_device_amps(n, CFG2["open"], fixed, amps.data_ptr(), k, direct_seed=direct)
            if best is None or st["device_ms"] < best["device_ms"]:
                best = st
        gbs = best["bytes"] / (best["device_ms"] * 1e-3) / 1e9
        out[name] = {"device_ms": best["device_ms"], "bytes": best["bytes"], "gbs": gbs, "frac_of_hbm": gbs / hbm_peak,
                     "candidates_kept": best["candidates_kept"], "fast_path": best["fast_path"]}
    return {"config": f"M=2^20 groups, l=6 (64 Mi candidates), synthetic Gaussian amplitudes in HBM; best of 5",
            "hbm_peak_gbs": hbm_peak, **out}


def xeb_cfg1(pb):
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
    approx.sync("f64")
    top, direct, _ = pb.api.postprocess_device_amps(n, list(range(l)), fixed, acc.data_ptr(), k,
                                                    direct_seed=pb.split_next(1, 0xD1EC7))
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
    exact ones up to the storage precision) -> the fused post-processing call
    (top-k with k = M, the paper's k = #groups, one direct sample per group, and
    both XEBs reduced on the device from the statevector)."""
    import numpy as np
    import torch
    n, l, M = 30, 6, len(fixed)
    P = 1 << l
    state = torch.empty(1 << n, dtype=torch.complex128, device="cuda")
    t0 = time.perf_counter()
    p.exact_state_device(state.data_ptr())
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    acc = torch.zeros(M * P * 2, dtype=torch.float64, device="cuda")
    for s0 in range(0, p.n_slices, 8):
        p.contract_groups_device(fixed, acc.data_ptr(), precision=precision, configs=None, slices=(s0, s0 + 8),
                                 sync=False)
    p.sync(precision)
    top, direct, st = pb.api.postprocess_device_amps(n, CFG2["open"], fixed, acc.data_ptr(), M,
                                                     direct_seed=pb.split_next(1, 0xD1EC7), d_state=state.data_ptr())
    t2 = time.perf_counter()
    cand = np.array([pb.member(n, CFG2["open"], int(f), i) for f in fixed for i in range(P)], np.int64)
    ex = state[torch.as_tensor(cand, device="cuda")].cpu().numpy()
    del state
    torch.cuda.empty_cache()
    ap = acc.cpu().numpy().view(np.complex128).reshape(-1)
    fid = abs(np.vdot(ex, ap)) ** 2 / (np.vdot(ap, ap).real * np.vdot(ex, ex).real)
    return {"config": f"cfg2 grid(5,6) n=30 cycles=14 l=6 M={M} K=0, all 256 slices, {precision}",
            # Porter-Thomas: keeping the top fraction k / (M 2^l) of exact probabilities gives XEB = ln(M 2^l / k)
            "xeb_topk": st["xeb_topk"], "k": M, "predicted_topk_exact": float(np.log(M * P / M)),
            "xeb_direct": st["xeb_direct"], "amplitude_fidelity_vs_exact": float(fid),
            "contract_and_sample_s": t2 - t1, "statevector_s": t1 - t0,
            "postprocess_device_ms": st["device_ms"],
            "note": "ideal probabilities from the GPU statevector (simulate_exact, bit-exact with the reference); "
                    "XEB reduced on the device by rcsg_postprocess"}


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    import paper_2406_18889_b200 as pb

    torch.cuda.set_device(local)
    pb.api.set_device(local)
    if world > 1:
        # stdout carries exactly one JSON line: no NCCL version banner
        if os.environ.get("NCCL_DEBUG", "").upper() in ("", "VERSION"):
            os.environ["NCCL_DEBUG"] = "WARN"
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    hbm_peak, bf16_peak, peak_kind = peaks()

    p = pb.Problem(CFG2["n"], CFG2["cycles"], CFG2["topology"], CFG2["seed"], CFG2["open"], CFG2["budget"],
                   CFG2["effort"]).build()
    assert p.n_slices == 256, p.n_slices
    M = args.groups
    fixed, dups = pb.build_candidate_set(30, CFG2["open"], M, pb.split_next(1, 0xCA11D))

    clocks = Clocks(local)
    head = measure(pb, p, fixed, args.precision, args, rank, world, clocks)
    clk = clocks.stop()
    alt = None
    if args.alt_precision != "none" and args.alt_precision != args.precision:
        a = measure(pb, p, fixed, args.alt_precision, args, rank, world)
        alt = {"value": a["value"], "unit": UNIT, "ms_per_step": a["ms_max"] / args.steps,
               "dtype": DTYPES[args.alt_precision], "gpu_launches": a["launches"],
               "complex_tflops_executed": a["exec_flops"] * world / (a["ms_max"] * 1e-3) / 1e12,
               "complex_tflops_reference_equivalent": a["plan_flops"] * world / (a["ms_max"] * 1e-3) / 1e12,
               "roofline": a["roofline"], "kernel_breakdown_ms": a["breakdown"]}
        del a

    e2e = cold = None
    if not args.no_e2e:
        e2e = e2e_warm(p, fixed, args.precision, head, world)
        if world == 1:
            cold = e2e_cold(pb, args.precision, M, e2e["value"])

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            smp = reference_sample(max(16, threads), threads, CFG2["budget"], M)
            cval, sample = reference_line_fields(smp, M)
            cpu = {"value": cval, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample}
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    scale = {}
    if rank == 0 and world == 1 and args.scale_configs != "none":
        for name in [c for c in args.scale_configs.split(",") if c]:
            try:
                alt_p = args.alt_precision if args.alt_precision != "none" else None
                if name == "cfg5":  # 60 qubits, 24 cycles: width 2^32 at a 2^38 B budget, 8 slices per mode
                    scale[name] = scale_bench(pb, name, args.precision, 8, budget_log2=38, alt=alt_p, alt_slices=8,
                                              trials=256, compare=True, replan=args.replan)
                else:
                    ns = args.cfg4_slices if name == "cfg4" else 64
                    scale[name] = scale_bench(pb, name, args.precision, ns, alt=alt_p, replan=args.replan)
            except Exception as e:  # pragma: no cover
                scale[name] = {"error": str(e)}

    post = None
    if rank == 0 and not args.no_post:
        try:
            post = post_bench(pb, hbm_peak)
        except Exception as e:  # pragma: no cover
            post = {"error": str(e)}

    xeb = None
    if rank == 0 and not args.no_xeb:
        try:
            xeb = {"cfg1": xeb_cfg1(pb)}
        except Exception as e:  # pragma: no cover
            xeb = {"cfg1": {"error": str(e)}}
        if world == 1:
            try:
                xeb["cfg2"] = xeb_cfg2(pb, p, fixed, args.precision)
            except Exception as e:  # pragma: no cover
                xeb["cfg2"] = {"error": str(e)}

    if rank == 0:
        ms_max = head["ms_max"]
        line = {
            "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": DTYPES[args.precision],
            "data": "synthetic (random circuit of the named shape)",
            "config": config_of(M),
            "precision": args.precision, "duplicate_groups": int(dups), "slices_per_call": head["S"],
            "l2": f"flushed between timed steps (256 MiB write, outside the per-step events); arena "
                  f"{head['arena'] / 2**30:.2f} GiB per GPU",
            "parallelism": f"slice-sharded x{world}",
            "group_slice_pairs_per_s": head["value"] * M,
            "complex_tflops_executed": head["exec_flops"] * world / (ms_max * 1e-3) / 1e12,
            "complex_tflops_reference_equivalent": head["plan_flops"] * world / (ms_max * 1e-3) / 1e12,
            "gpu_launches": head["launches"],
            "roofline": head["roofline"],
            "kernel_breakdown_ms": head["breakdown"],
            "e2e": e2e, "e2e_cold": cold, "cpu_baseline": cpu, "clocks": clk,
            "postprocess": post, "xeb": xeb, "scale_configs": scale or None,
        }
        if alt:
            line[args.alt_precision] = alt
        emit(line)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.stdout.flush()
    _RESULT_FD = os.dup(1)
    os.dup2(2, 1)
    sys.exit(main())
