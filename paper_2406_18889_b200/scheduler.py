"""Slice scheduler: shards the independent slices of a plan across the GPUs of
one box (one process per GPU, torch.distributed / NCCL) and combines the
partial amplitude tensors with one collective.

Determinism (the reference guarantees bit-identical results for any worker
count, test_contraction.cpp:84-93): the slice range is cut into
``N_BLOCKS`` canonical contiguous blocks independent of the world size; each
block is summed on one GPU in ascending slice order into its own [M][2^l]
partial, the partials are all-gathered (the path's only exchange step, sent
over NVLink by NCCL), and every rank adds them in block order.  So the result
is bit-identical for 1, 2, 4 or 8 GPUs.

The block contraction itself is injected (``contract_block``), so the same
host logic runs the GPU path (``gpu_block_fn``) and, in the CPU tests, the
oracle (gloo, world size 2).
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


def contract_sharded(contract_block: Callable[[int, int], np.ndarray], n_slices: int, rank: int = 0,
                     world: int = 1, group=None, n_blocks: int = N_BLOCKS) -> np.ndarray:
    """Amplitudes summed over all slices, identical on every rank.

    contract_block(s0, s1) -> complex array [M][2^l] summed over slices s0..s1-1 (ascending).
    """
    blocks = slice_blocks(n_slices, n_blocks)
    mine = blocks_of_rank(len(blocks), rank, world)
    partials = {b: np.asarray(contract_block(*blocks[b]), np.complex128) for b in mine}
    shape = next(iter(partials.values())).shape if partials else None
    if world > 1:
        import torch
        import torch.distributed as dist
        if shape is None:
            raise RuntimeError("every rank needs at least one block (world size > block count)")
        local = np.stack([partials[b] for b in mine]).view(np.float64)
        per_rank = [len(blocks_of_rank(len(blocks), r, world)) for r in range(world)]
        maxb = max(per_rank)
        buf = np.zeros((maxb,) + local.shape[1:], np.float64)
        buf[:len(mine)] = local
        t = torch.from_numpy(buf)
        if dist.get_backend(group) == "nccl":
            t = t.cuda()
        gathered = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(gathered, t, group=group)
        for r in range(world):
            got = gathered[r].cpu().numpy()
            for j, b in enumerate(blocks_of_rank(len(blocks), r, world)):
                partials[b] = got[j].view(np.complex128)
    total = np.zeros_like(partials[0])
    for b in range(len(blocks)):  # fixed block order
        total = total + partials[b]
    return total


def gpu_block_fn(problem, fixed, precision: str = "tf32", configs=None):
    """contract_block for the GPU path: a fresh device accumulator per block."""
    import torch

    P = 1 << problem.n_open

    def run(s0: int, s1: int) -> np.ndarray:
        acc = torch.zeros(len(fixed) * P * 2, dtype=torch.float64, device="cuda")
        problem.contract_groups_device(fixed, acc.data_ptr(), precision=precision, configs=configs,
                                       slices=(s0, s1))
        return acc.cpu().numpy().view(np.complex128).reshape(len(fixed), P)

    return run
