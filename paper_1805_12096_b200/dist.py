"""Multi-GPU driver: one process per GPU, torch.distributed (NCCL) for plumbing only.

Sentences are independent (static quantization scales), so the decode
path has no exchange step: each rank decodes its own shard with libmnmt and the only
collective is the final gather of output ids to rank 0 (A11).
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np


def shard_round_robin(lengths: np.ndarray, rank: int, world: int) -> np.ndarray:
    """Strong-scaling shard of one sentence set: globally sort by length (stable), deal
    positions r, r+G, ... to rank r, so every rank gets the same length mix."""
    order = np.argsort(np.asarray(lengths), kind="stable")
    return order[rank::world].astype(np.int64)


def pack_ids(outs: List[np.ndarray], max_len: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """Flat [sum max_len] id buffer (layout of mnmt_translate) + lengths."""
    offs = np.concatenate([[0], np.cumsum(max_len)]).astype(np.int64)
    flat = np.zeros(int(offs[-1]), np.int32)
    lens = np.zeros(len(outs), np.int32)
    for i, o in enumerate(outs):
        flat[offs[i]:offs[i] + len(o)] = o
        lens[i] = len(o)
    return flat, lens


def gather_ids(ids, lens, group=None):
    """All-gather every rank's (flat ids, lengths) tensors; returns per-rank lists on all ranks.

    Works for any backend: NCCL with CUDA tensors, gloo with CPU tensors.  Sizes differ per
    rank, so counts are exchanged first and buffers are padded to the maximum."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = ids.device
    cnt = torch.tensor([ids.numel(), lens.numel()], dtype=torch.int64, device=dev)
    cnts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(cnts, cnt, group=group)
    mi = max(int(c[0]) for c in cnts)
    ml = max(int(c[1]) for c in cnts)
    pid = torch.zeros(max(mi, 1), dtype=ids.dtype, device=dev)
    pid[:ids.numel()] = ids
    pln = torch.zeros(max(ml, 1), dtype=lens.dtype, device=dev)
    pln[:lens.numel()] = lens
    gi = [torch.zeros_like(pid) for _ in range(world)]
    gl = [torch.zeros_like(pln) for _ in range(world)]
    dist.all_gather(gi, pid, group=group)
    dist.all_gather(gl, pln, group=group)
    return ([g[:int(c[0])] for g, c in zip(gi, cnts)], [g[:int(c[1])] for g, c in zip(gl, cnts)])


def unshard(per_rank_outs: List[List[np.ndarray]], shards: List[np.ndarray], n: int) -> List[np.ndarray]:
    """Restore input order from strong-scaling shards."""
    res: List[np.ndarray] = [None] * n  # type: ignore
    for outs, idx in zip(per_rank_outs, shards):
        for o, i in zip(outs, idx):
            res[int(i)] = o
    return res
