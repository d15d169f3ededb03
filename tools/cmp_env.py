"""Contract one cfg4 slice (M groups, tf32) and save the amplitudes (argv[1]); with
argv[2] also compare against an earlier file: norm-relative difference per group.
Used to check a kernel-selection knob (env) against the default on the same inputs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2406_18889_b200 as pb
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
M = int(os.environ.get("M", "64"))
p = pb.Problem(53, 20, "sycamore53", 1, list(range(6)), 1 << 36, "low").build(
    plan_json=open(os.path.join(root, "plans", "cfg4.json")).read())
fixed, _ = pb.build_candidate_set(53, list(range(6)), M, pb.split_next(1, 0xca11d))
a = p.contract_groups(fixed, precision="tf32", configs=None, slices=(0, 1))
np.save(sys.argv[1], a)
if len(sys.argv) > 2:
    b = np.load(sys.argv[2])
    e = np.linalg.norm(a - b, axis=1) / np.maximum(np.linalg.norm(b, axis=1), 1e-300)
    print("max norm-rel diff", float(e.max()), "bitwise", bool(np.array_equal(a, b)))
