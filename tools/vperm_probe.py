"""Shared-operand variant order (RCSG_NO_VPERM) on the committed cfg3 / cfg4 plans:
one slice at tf32, M = 64, with and without; the results must be bit-identical."""
import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2406_18889_b200 as pb
CF = {"cfg3": (53, 12, "sycamore53", 36), "cfg4": (53, 20, "sycamore53", 36)}
for name, M in (("cfg3", 64), ("cfg4", 64)):
    n, m, topo, blog = CF[name]
    p = pb.Problem(n, m, topo, 1, list(range(6)), 1 << blog, "low").build(plan_json=open(f"plans/{name}.json").read())
    fixed, _ = pb.build_candidate_set(n, list(range(6)), M, pb.split_next(1, 0xCA11D))
    out = {}
    for nf in ("0", "1"):
        if nf == "1": os.environ["RCSG_NO_VPERM"] = "1"
        else: [os.environ.pop(x, None) for x in ("RCSG_NO_VPERM",)]
        p.release()
        out[nf] = p.contract_groups(fixed, precision="tf32", configs=None, slices=(0, 1))
    p.release()
    e = np.linalg.norm(out["0"] - out["1"], axis=1) / np.linalg.norm(out["1"], axis=1)
    print(name, "vperm vs none max norm-rel", float(e.max()), "identical", bool(np.array_equal(out["0"], out["1"])), flush=True)
