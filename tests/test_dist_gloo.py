"""The N > 1 path of bench.py on CPU: world_size 2 over gloo (127.0.0.1).

Each rank runs the functions bench.py runs (paper_1805_12096_b200.dist): its shard of the set
(strong: length-sorted round-robin; weak: its own set), a decode of that shard, the flat id
layout of mnmt_translate, the padded all_gather, and on rank 0 the unshard plan that
mnmt_op_gather_rows executes on the GPU (here its numpy twin `unshard_host`).  The decode of a
shard is the CPU oracle (test infrastructure: libmnmt needs a GPU); the job's ids in input
order must equal the oracle's decode of the whole set.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle.oracle as O
import synth
from paper_1805_12096_b200 import dist as D

DIMS = synth.ModelDims("gloo-tiny", 32, 64, 4, vocab=64, enc_layers=1, dec_layers=2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _set(seed):
    return synth.random_set(61, 1, 23, seed=seed, vocab=DIMS.vocab)


def _worker(rank, world, port, scaling, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        om = O.OracleModel(DIMS, synth.make_weights(DIMS, seed=3))
        if scaling == "strong":
            full = _set(40)
            shards = [D.shard_round_robin(full.lengths, r, world) for r in range(world)]
            local, idx = D.local_set(full, rank, world, "strong")
            assert np.array_equal(idx, shards[rank])
            ml_all = full.max_len
        else:
            local, idx = D.local_set(_set(40 + rank), rank, world, "weak")
            assert idx is None
            shards = [np.arange(r * local.n, (r + 1) * local.n) for r in range(world)]
            ml_all = np.concatenate([_set(40 + r).max_len for r in range(world)])
        plan = D.gather_plan(ml_all, shards)
        outs = om.decode_many(local, 1)                 # stands in for the GPU decode
        flat, lens = D.pack_ids(outs, local.max_len)
        gi, gl = D.all_gather_padded(torch.from_numpy(flat), torch.from_numpy(lens), plan)
        if rank == 0:
            ids, ln = D.unshard_host(gi.numpy(), gl.numpy(), plan)
            got = D.split_rows(ids, ln, ml_all)
            if scaling == "strong":
                ref = om.decode_many(_set(40), 1)
            else:
                ref = sum((om.decode_many(_set(40 + r), 1) for r in range(world)), [])
            q.put((len(got) == len(ref)) and all(np.array_equal(a, b) for a, b in zip(got, ref)))
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


def test_gather_plan_host_roundtrip():
    """Unshard plan on one process: a random 3-way split of ragged rows comes back in order."""
    rng = np.random.default_rng(0)
    ml = rng.integers(0, 9, size=50)
    outs = [rng.integers(3, 99, size=rng.integers(0, m + 1)).astype(np.int32) for m in ml]
    perm = rng.permutation(50)
    shards = [perm[:17], perm[17:20], perm[20:]]
    plan = D.gather_plan(ml, shards)
    gi = np.zeros(plan.world * plan.id_cap, np.int32)
    gl = np.zeros(plan.world * plan.n_cap, np.int32)
    for r, s in enumerate(shards):
        f, l = D.pack_ids([outs[i] for i in s], ml[s])
        gi[r * plan.id_cap:r * plan.id_cap + len(f)] = f
        gl[r * plan.n_cap:r * plan.n_cap + len(l)] = l
    ids, ln = D.unshard_host(gi, gl, plan)
    got = D.split_rows(ids, ln, ml)
    assert all(np.array_equal(a, b) for a, b in zip(got, outs))


@pytest.mark.timeout(300)
@pytest.mark.parametrize("scaling", ["strong", "weak"])
def test_bench_multi_rank_path_gloo_world2(scaling):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, scaling, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=10) is True
