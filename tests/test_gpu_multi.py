"""Multi-GPU slice scheduler over NCCL (one process per GPU): the slice-summed
amplitudes are bit-identical on every rank and equal to the single-GPU result.
Needs >= 2 GPUs (skipped otherwise; the host logic is covered with gloo in
test_scheduler.py)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _worker(rank, world, port_no, q):
    import torch
    import torch.distributed as dist
    import paper_2406_18889_b200 as pb
    from paper_2406_18889_b200 import scheduler
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    torch.cuda.set_device(rank)
    pb.api.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        p = pb.Problem(10, 10, "line", 17, [0, 3, 5, 8], 20000, "low").build()
        fixed = np.array([0, 5, 22, 63], np.uint64)
        out = scheduler.contract_sharded(scheduler.gpu_block_fn(p, fixed, "tf32"), p.n_slices, rank, world)
        assert out.is_cuda  # partials and their sum stay on the device
        q.put((rank, out.cpu().numpy().view(np.float64).tobytes()))
    finally:
        dist.destroy_process_group()


def test_two_gpu_scheduler_bit_identical():
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    import multiprocessing as mp
    import paper_2406_18889_b200 as pb
    from paper_2406_18889_b200 import scheduler
    p = pb.Problem(10, 10, "line", 17, [0, 3, 5, 8], 20000, "low").build()
    fixed = np.array([0, 5, 22, 63], np.uint64)
    single = scheduler.contract_sharded(scheduler.gpu_block_fn(p, fixed, "tf32"), p.n_slices, 0, 1).cpu().numpy()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port_no = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port_no, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    for r in range(2):
        got = np.frombuffer(res[r], np.float64).view(np.complex128).reshape(single.shape)
        assert np.array_equal(got, single)
