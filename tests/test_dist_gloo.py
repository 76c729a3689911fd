"""Multi-process host logic of the N>1 path on CPU: world_size 2 over gloo (127.0.0.1)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from paper_1805_12096_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _fake_decode(ss, idx):
    # stands in for libmnmt on CPU: a deterministic, length-varying id sequence per sentence
    out = []
    for i in idx:
        src = ss.ids[ss.offsets[i]:ss.offsets[i + 1]]
        out.append((src[: max(0, int(ss.max_len[i]) - (int(i) % 3))] * 7 + int(i)) % 36000)
    return out


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ss = synth.newstest_set()
        idx = D.shard_round_robin(ss.lengths, rank, world)
        outs = _fake_decode(ss, idx)
        flat, lens = D.pack_ids(outs, ss.max_len[idx])
        gi, gl = D.gather_ids(torch.from_numpy(flat), torch.from_numpy(lens))
        if rank == 0:
            per_rank = []
            shards = []
            for r in range(world):
                ml = ss.max_len[D.shard_round_robin(ss.lengths, r, world)]
                offs = np.concatenate([[0], np.cumsum(ml)])
                f, l = gi[r].numpy(), gl[r].numpy()
                per_rank.append([f[offs[k]:offs[k] + l[k]] for k in range(len(l))])
                shards.append(D.shard_round_robin(ss.lengths, r, world))
            res = D.unshard(per_rank, shards, ss.n)
            ref = _fake_decode(ss, range(ss.n))
            q.put(all(np.array_equal(a, b) for a, b in zip(res, ref)))
    finally:
        dist.destroy_process_group()


def test_shard_partition_and_balance():
    L = synth.newstest_lengths()
    for G in (1, 2, 4, 8):
        shards = [D.shard_round_robin(L, r, G) for r in range(G)]
        allidx = np.sort(np.concatenate(shards))
        assert np.array_equal(allidx, np.arange(len(L)))
        words = [int(L[s].sum()) for s in shards]
        assert max(words) - min(words) <= 100     # same length mix on every rank


@pytest.mark.timeout(300)
def test_gather_ids_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=10) is True
