"""Generates the golden fixtures in tests/golden/ from the UNMODIFIED reference
library (oracle/_ref/librcs_ref.so, built from /root/reference/proj/src by
oracle/Makefile).  Run in the build container, where /root/reference exists:

    make -C oracle && python tests/golden/make_golden.py

Every fixture records the reference's own outputs (plans, amplitudes, sampler
picks) for the BASELINE configs' small cases, so the checker (oracle/port) and
the GPU path can be pinned on a box without the reference sources.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref  # noqa: E402

CASES = {
    # name: (n, cycles, topology, seed, open, budget, effort, K, m)
    "cfg1": (12, 8, "grid(3,4)", 1, [0, 1, 2], 1 << 30, "low", 0, 1),
    "sliced_line10": (10, 10, "line", 17, [0, 3, 5, 8], 20000, "low", 0, 1),
    "broken_ring10": (10, 10, "ring", 62, list(range(10)), 1 << 30, "low", 5, 16),
    "grid44_sliced_broken": (16, 10, "grid(4,4)", 3, [0, 1, 2, 3], 1 << 18, "low", 3, 5),
}


def problem_fixture(name, spec, n_groups):
    p = ref.RefProblem(*spec).build()
    n, l = spec[0], len(spec[4])
    if n > l:
        fixed, dup = ref.candidates(n, spec[4], n_groups, ref.split_next(spec[3], 0xCA11D))
    else:
        fixed, dup = np.zeros(1, np.uint64), 0
    amps = np.stack([p.contract_group(int(g)) for g in fixed])
    out = dict(spec=np.array(repr(spec)), group_fixed=fixed, duplicate_groups=dup, amplitudes=amps,
               gates=p.gates(), steps=p.plan["steps"], sliced=p.plan["sliced"], broken=p.plan["broken"],
               fixed_outputs=p.plan["fixed_outputs"], configs=p.plan["configs"],
               totals=np.array([p.plan["flops_per_slice"], p.plan["traffic_bytes_per_slice"],
                                p.plan["peak_bytes"], p.plan["memory_budget_bytes"]], np.uint64),
               leaf_rank=p.net["leaf_rank"], leaf_labels=p.net["leaf_labels"], leaf_data=p.net["leaf_data"],
               output_labels=p.net["output_labels"], open_labels=p.net["open_labels"],
               open_qubits=p.net["open_qubits"], n_labels=p.net["n_labels"],
               label_names=np.array(p.net["label_names"]))
    if n <= 16:
        out["statevector"] = p.exact(cap=16)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, amps.shape, len(p.plan["steps"]), "steps", len(p.plan["sliced"]), "sliced")


def sampler_fixture():
    rng = np.random.default_rng(7)
    n, open_q = 12, [0, 1, 2]
    fixed, dup = ref.candidates(n, open_q, 512, ref.split_next(1, 0xCA11D))
    # the reference's ProbFn is a function of the bitstring index: duplicate
    # groups see identical probabilities
    table = rng.exponential(size=1 << n) / 4096
    probs = np.array([[table[ref.member(n, open_q, int(f), i)] for i in range(8)] for f in fixed])
    ties = np.full((64, 8), 1.0 / 512)
    fixed_t, _ = ref.candidates(9, [1, 4, 7], 64, 5)
    ks = np.array([1, 7, 64, 512, 4096])
    topk = {f"topk_{k}": ref.top_k(n, open_q, fixed, probs, int(k)) for k in ks}
    tie = {f"ties_{k}": ref.top_k(9, [1, 4, 7], fixed_t, ties, int(k)) for k in (1, 100, 512)}
    seed = ref.split_next(1, 0xD1EC7)
    direct = ref.direct(n, open_q, fixed, probs, seed)
    q = rng.exponential(size=1000) / 4096
    xeb = ref.xeb(12, np.arange(1000, dtype=np.uint64), q)
    lex = np.array([[i, ref.lexkey(i, 12)] for i in (0, 1, 8, 6, 4095, 1234)], np.uint64)
    np.savez_compressed(os.path.join(HERE, "sampler.npz"), fixed=fixed, duplicate_groups=dup, probs=probs,
                        ties=ties, fixed_ties=fixed_t, direct_seed=np.uint64(seed), direct=direct, q=q, xeb=xeb,
                        lexkeys=lex, split_ca11d=np.uint64(ref.split_next(1, 0xCA11D)),
                        split_d1ec7=np.uint64(seed), **topk, **tie)
    print("sampler fixtures")


if __name__ == "__main__":
    for name, spec in CASES.items():
        problem_fixture(name, spec, 64 if name == "cfg1" else 8)
    sampler_fixture()
