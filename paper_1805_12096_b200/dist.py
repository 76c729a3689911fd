"""Multi-GPU driver: one process per GPU, torch.distributed (NCCL) for plumbing only.

Sentences are independent (static quantization scales), so the decode
path has no exchange step:

* weak scaling: every rank decodes its own newstest-shaped set;
* strong scaling: one set is globally length-sorted and dealt round-robin, so every rank gets
  the same length mix and forms its own word-budget batches.

The only collective is the final gather of output ids (A11): one all_gather of the padded
per-rank id buffers and lengths, then -- strong scaling -- the rows are put back in input
order on rank 0 by libmnmt's `mnmt_op_gather_rows` (device) or `unshard_host` (the same
plan, numpy; used by the CPU tests).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Tuple

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


@dataclass
class GatherPlan:
    """Static layout of one all_gather of per-rank (flat ids, lengths) and of the unshard.

    Rank r's flat ids (mnmt_translate layout over its rows) land at r * id_cap of the gathered
    id buffer, its lengths at r * n_cap of the gathered length buffer.  For source row
    i = r * n_cap + k (k < n_cap; rows beyond a rank's count are zero-length padding):
    src_off[i] = r * id_cap + (prefix sum of that rank's max_len)[k], dst_row[i] = the
    sentence's index in the input (padding rows: the scratch row n), dst_off = prefix sum of
    max_len in input order (+ one scratch row)."""
    world: int
    n: int                  # sentences in input order
    id_cap: int
    n_cap: int
    src_off: np.ndarray     # int64 [world * n_cap]
    dst_row: np.ndarray     # int32 [world * n_cap]
    dst_off: np.ndarray     # int64 [n + 1]
    out_total: int          # sum max_len (dst_off[n])


def gather_plan(max_len: np.ndarray, shards: List[np.ndarray]) -> GatherPlan:
    """Plan for shards[r] = input indices of rank r's rows (in that rank's row order)."""
    max_len = np.asarray(max_len, np.int64)
    world, n = len(shards), len(max_len)
    n_cap = max(1, max(len(s) for s in shards))
    id_cap = max(1, max(int(max_len[s].sum()) for s in shards))
    src_off = np.zeros(world * n_cap, np.int64)
    dst_row = np.full(world * n_cap, n, np.int32)
    for r, s in enumerate(shards):
        lo = np.concatenate([[0], np.cumsum(max_len[s])[:-1]]).astype(np.int64) if len(s) else np.zeros(0, np.int64)
        src_off[r * n_cap:r * n_cap + len(s)] = r * id_cap + lo
        dst_row[r * n_cap:r * n_cap + len(s)] = s
    dst_off = np.zeros(n + 1, np.int64)
    np.cumsum(max_len, out=dst_off[1:])
    return GatherPlan(world, n, id_cap, n_cap, src_off, dst_row, dst_off, int(dst_off[n]))


def all_gather_padded(ids, lens, plan: GatherPlan, group=None):
    """One all_gather of the padded id buffer and one of the lengths (NCCL: CUDA tensors;
    gloo: CPU tensors).  Returns (ids [world * id_cap], lens [world * n_cap])."""
    import torch
    import torch.distributed as dist
    pid = torch.zeros(plan.id_cap, dtype=ids.dtype, device=ids.device)
    pid[:ids.numel()] = ids
    pln = torch.zeros(plan.n_cap, dtype=lens.dtype, device=lens.device)
    pln[:lens.numel()] = lens
    gi = torch.empty(plan.world * plan.id_cap, dtype=ids.dtype, device=ids.device)
    gl = torch.empty(plan.world * plan.n_cap, dtype=lens.dtype, device=lens.device)
    dist.all_gather_into_tensor(gi, pid, group=group)
    dist.all_gather_into_tensor(gl, pln, group=group)
    return gi, gl


def unshard_host(gids: np.ndarray, glens: np.ndarray, plan: GatherPlan):
    """The unshard of mnmt_op_gather_rows in numpy (CPU tests): (flat ids in input order,
    lengths in input order)."""
    out = np.zeros(plan.out_total + 1, np.int32)
    ln = np.zeros(plan.n + 1, np.int32)
    for i in range(plan.world * plan.n_cap):
        r, L = int(plan.dst_row[i]), int(glens[i])
        out[plan.dst_off[r]:plan.dst_off[r] + L] = gids[plan.src_off[i]:plan.src_off[i] + L]
        ln[r] = L
    return out[:plan.out_total], ln[:plan.n]


class DeviceUnshard:
    """The unshard on rank 0's GPU: plan arrays uploaded once, mnmt_op_gather_rows per call."""

    def __init__(self, plan: GatherPlan, device):
        import torch
        self.plan = plan
        self.src_off = torch.from_numpy(plan.src_off).to(device)
        self.dst_row = torch.from_numpy(plan.dst_row).to(device)
        dst_off = np.concatenate([plan.dst_off, [plan.out_total]]).astype(np.int64)  # + scratch
        self.dst_off = torch.from_numpy(dst_off).to(device)
        self.out = torch.zeros(plan.out_total + 1, dtype=torch.int32, device=device)
        self.lens = torch.zeros(plan.n + 1, dtype=torch.int32, device=device)

    def __call__(self, gids, glens, stream=None):
        from . import mnmt as M
        M.op_gather_rows(gids.data_ptr(), self.src_off.data_ptr(), glens.data_ptr(),
                         self.dst_row.data_ptr(), self.dst_off.data_ptr(),
                         self.plan.world * self.plan.n_cap, self.out.data_ptr(),
                         self.lens.data_ptr(), stream)
        return self.out[:self.plan.out_total], self.lens[:self.plan.n]


def split_rows(flat: np.ndarray, lens: np.ndarray, max_len: np.ndarray) -> List[np.ndarray]:
    """Per-sentence id arrays from the mnmt_translate layout."""
    offs = np.concatenate([[0], np.cumsum(max_len)]).astype(np.int64)
    return [flat[offs[i]:offs[i] + int(lens[i])] for i in range(len(lens))]


def local_set(sset, rank: int, world: int, scaling: str, weak_seed: Optional[int] = None):
    """The rows rank `rank` decodes: (its sentence set, input indices or None).
    weak: `sset` itself (each rank builds its own set, seed weak_seed + rank, outside);
    strong: the round-robin shard of `sset`."""
    if scaling == "weak" or world == 1:
        return sset, None
    idx = shard_round_robin(sset.lengths, rank, world)
    return sset.subset(idx), idx
