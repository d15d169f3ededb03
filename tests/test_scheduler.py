"""Multi-GPU slice scheduler host logic on CPU: canonical block sharding and the
deterministic all-gather + ordered sum, run with torch.distributed gloo at
world size 2 (the block contraction is the CPU oracle here; on GPUs it is the
device path).  Results must be bit-identical for any world size and equal to
the full contraction."""
import os
import socket

import numpy as np
import pytest

from paper_2406_18889_b200 import scheduler

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_blocks_partition_slices():
    for n in (1, 2, 7, 8, 256):
        blocks = scheduler.slice_blocks(n)
        covered = [s for a, b in blocks for s in range(a, b)]
        assert covered == list(range(n))
    for world in (1, 2, 3, 4, 8):
        owned = sorted(b for r in range(world) for b in scheduler.blocks_of_rank(8, r, world))
        assert owned == list(range(8))


def _oracle_block_fn():
    from oracle import port
    g = dict(np.load(os.path.join(GOLDEN, "sliced_line10.npz")))
    net = dict(leaf_rank=g["leaf_rank"], leaf_labels=g["leaf_labels"], leaf_data=g["leaf_data"],
               n_labels=int(g["n_labels"]), n_qubits=len(g["output_labels"]), output_labels=g["output_labels"],
               open_labels=g["open_labels"], open_qubits=g["open_qubits"])
    pn = port.PortNet(net, dict(steps=g["steps"], sliced=g["sliced"], broken=g["broken"]))
    fixed = g["group_fixed"]

    def block(s0, s1):
        return np.stack([pn.contract_group(int(f), slices=(s0, s1)) for f in fixed])

    return block, 1 << len(g["sliced"]), g["amplitudes"]


def _worker(rank, world, port_no, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        block, n_slices, _ = _oracle_block_fn()
        out = scheduler.contract_sharded(block, n_slices, rank, world)
        q.put((rank, out.view(np.float64).tobytes()))
    finally:
        dist.destroy_process_group()


def test_world2_gloo_bit_identical_to_world1():
    from oracle import port
    if not port.available():
        pytest.skip("oracle port not built")
    import multiprocessing as mp
    block, n_slices, ref_amps = _oracle_block_fn()
    single = scheduler.contract_sharded(block, n_slices, 0, 1)
    # the slice sum equals the full contract_group of the reference (different order -> fp tolerance)
    assert np.max(np.abs(single - ref_amps)) <= 1e-12 * np.max(np.abs(ref_amps))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port_no = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port_no, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        got = np.frombuffer(res[r], np.float64).view(np.complex128).reshape(single.shape)
        assert np.array_equal(got, single)
