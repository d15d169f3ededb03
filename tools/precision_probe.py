"""Amplitude error per precision mode at scale: one slice of the committed
cfg3 / cfg4 / cfg5 plans (plans/<cfg>.json), M groups, contracted in every
mode; errors are norm-relative per group against the f64 SIMT mode (which is
pinned to the reference's CPU executor at small sizes by the parity tests), or
the fp32 SIMT mode where the f64 arena does not fit (cfg5).  RCSG_TF32_CHOP=1:
tf32 operands reach the MMA unrounded (its own truncation).
Env: CFGS (default cfg3,cfg4,cfg5), M (default 8), SLICE (default 0),
PRECS (default tf32,f16,bf16).  One JSON line per config."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2406_18889_b200 as pb  # noqa: E402

CFGS = {"cfg3": (53, 12, "sycamore53", 36), "cfg4": (53, 20, "sycamore53", 36), "cfg5": (60, 24, "zuchongzhi60", 38)}
M = int(os.environ.get("M", "8"))
S = int(os.environ.get("SLICE", "0"))
for name in os.environ.get("CFGS", "cfg3,cfg4,cfg5").split(","):
    n, m, topo, blog = CFGS[name]
    p = pb.Problem(n, m, topo, 1, list(range(6)), 1 << blog, "low").build(
        plan_json=open(os.path.join(ROOT, "plans", f"{name}.json")).read())
    fixed, _ = pb.build_candidate_set(n, list(range(6)), M, pb.split_next(1, 0xCA11D))
    res, secs = {}, {}
    anchor = "f64"
    for prec in ["f64"] + os.environ.get("PRECS", "tf32,f16,bf16").split(","):
        t = time.time()
        try:
            res[prec] = p.contract_groups(fixed, precision=prec, configs=None, slices=(S, S + 1))
        except pb.api.CapacityError:  # the f64 arena does not fit: fp32 SIMT (f32) is the anchor
            p.release()
            anchor = "f32"
            res[anchor] = p.contract_groups(fixed, precision="f32", configs=None, slices=(S, S + 1))
        secs[prec if prec in res else anchor] = time.time() - t
        p.release()
    ref = res[anchor]
    nrm = np.maximum(np.linalg.norm(ref, axis=1), 1e-300)
    out = {"cfg": name, "groups": M, "slice": S, "steps": len(p.plan["steps"]), "anchor": anchor,
           "tf32_chop": bool(os.environ.get("RCSG_TF32_CHOP")), "seconds": secs}
    for prec, a in res.items():
        if prec == anchor:
            continue
        e = np.linalg.norm(a - ref, axis=1) / nrm
        out[prec] = {"max_norm_rel": float(e.max()), "median_norm_rel": float(np.median(e))}
    print(json.dumps(out), flush=True)
