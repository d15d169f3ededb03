"""Slice scheduler: shards the independent slices of a plan across the GPUs of
one box (one process per GPU, torch.distributed / NCCL) and combines the
partial amplitude tensors with one collective.

Determinism (the reference guarantees bit-identical results for any worker
count, test_contraction.cpp:84-93): the slice range is cut into
``N_BLOCKS`` canonical contiguous blocks independent of the world size; each
block is summed on one GPU in ascending slice order into its own [M][2^l]
partial, the partials are all-gathered (the path's only exchange step, sent
over NVLink by NCCL) and every rank adds them in block order.  So the result
is bit-identical for 1, 2, 4 or 8 GPUs.

The partials stay where the block contraction leaves them: device tensors on
the GPU path (``gpu_block_fn``: NCCL gathers device memory and the ordered sum
runs on the device), host arrays in the CPU tests (gloo, world size 2, the
oracle as the block contraction).  The in-process C-ABI equivalent for one
process driving several GPUs is ``rcsg_multi_contract_groups`` (multi.cu).
"""
from __future__ import annotations

from typing import Callable

import numpy as np

N_BLOCKS = 8


def slice_blocks(n_slices: int, n_blocks: int = N_BLOCKS):
    """Canonical contiguous blocks [s0, s1) of the slice range (independent of world size)."""
    n_blocks = max(1, min(n_blocks, n_slices))
    edges = [n_slices * b // n_blocks for b in range(n_blocks + 1)]
    return [(edges[b], edges[b + 1]) for b in range(n_blocks)]


def blocks_of_rank(n_blocks: int, rank: int, world: int):
    """Round-robin assignment of canonical blocks to ranks."""
    return [b for b in range(n_blocks) if b % world == rank]


def _as_real_tensor(x):
    """A block partial as a float64 torch tensor [..., 2] (device or host), or the
    numpy array itself when torch is not in play."""
    import torch
    if isinstance(x, torch.Tensor):
        return torch.view_as_real(x) if x.is_complex() else x
    return torch.from_numpy(np.ascontiguousarray(x).view(np.float64).reshape(*x.shape, 2))


def contract_sharded(contract_block: Callable[[int, int], object], n_slices: int, rank: int = 0,
                     world: int = 1, group=None, n_blocks: int = N_BLOCKS):
    """Amplitudes summed over all slices, identical on every rank.

    contract_block(s0, s1) -> complex [M][2^l] summed over slices s0..s1-1
    (ascending): a numpy array, or a torch tensor (complex, or float64 with a
    trailing re/im axis) that may live on the GPU.  The result has the type of
    the partials (a device tensor stays on the device)."""
    blocks = slice_blocks(n_slices, n_blocks)
    mine = blocks_of_rank(len(blocks), rank, world)
    raw = {b: contract_block(*blocks[b]) for b in mine}
    if world == 1 and all(isinstance(v, np.ndarray) for v in raw.values()):
        total = np.zeros_like(raw[0])
        for b in range(len(blocks)):  # fixed block order
            total = total + raw[b]
        return total
    import torch
    import torch.distributed as dist
    partials = {b: _as_real_tensor(v) for b, v in raw.items()}
    if world > 1:
        if not partials:
            raise RuntimeError("every rank needs at least one block (world size > block count)")
        proto = next(iter(partials.values()))
        if dist.get_backend(group) == "nccl" and not proto.is_cuda:
            proto = proto.cuda()
            partials = {b: t.cuda() for b, t in partials.items()}
        maxb = max(len(blocks_of_rank(len(blocks), r, world)) for r in range(world))
        buf = torch.zeros((maxb,) + tuple(proto.shape), dtype=torch.float64, device=proto.device)
        for j, b in enumerate(mine):
            buf[j].copy_(partials[b])
        gathered = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(gathered, buf, group=group)  # the only exchange step (NVLink on NCCL)
        for r in range(world):
            for j, b in enumerate(blocks_of_rank(len(blocks), r, world)):
                partials[b] = gathered[r][j]
    total = partials[0].clone()
    for b in range(1, len(blocks)):  # fixed block order, on the partials' device
        total += partials[b]
    if all(isinstance(v, np.ndarray) for v in raw.values()):
        return total.cpu().numpy().view(np.complex128).reshape(total.shape[:-1])
    return torch.view_as_complex(total.contiguous())


def gpu_block_fn(problem, fixed, precision: str = "tf32", configs=None):
    """contract_block for the GPU path: a device accumulator per block (zeroed on
    torch's stream; the executor's stream waits for it), returned on the device."""
    import torch

    P = 1 << problem.n_open

    def run(s0: int, s1: int):
        acc = torch.zeros(len(fixed) * P * 2, dtype=torch.float64, device="cuda")
        problem.contract_groups_device(fixed, acc.data_ptr(), precision=precision, configs=configs,
                                       slices=(s0, s1))
        return acc.view(len(fixed), P, 2)

    return run
