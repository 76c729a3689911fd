"""Shortlist (F2) A/B on one B200: newstest-shaped small-AAN job, bench launch options, median of
5 timed jobs (device-resident ids) for
  plain      full-vocabulary argmax
  sl-full    MNMT_SHORTLIST with a frequent list = the whole vocabulary (union = V: isolates the
             cost of the masks, the gather and the per-job size read-back)
  sl-unif    the bench tables (100 + 100) with uniform source ids (the SURVEY recipe)
  sl-zipf    the same tables with Zipf(1.1) source ids (natural-text-like repetition: far fewer
             distinct source words per batch, so far smaller shortlists)
Prints one JSON line per variant with ms per job and the mean shortlist union size."""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1805_12096_b200 import mnmt as M  # noqa: E402

dims = synth.PRESETS[os.environ.get("PRESET", "small-aan")]
budget = int(os.environ.get("BUDGET", 8192))
m = M.Model(dims, synth.make_weights(dims, 1))
for k, v in [("max_concurrent_rows", 4096), ("lanes", 3), ("lane_tiers", 40), ("green_sms", 56),
             ("pers_reserve", 16)]:
    m.set_option(k, v)
base = synth.newstest_set(seed=2014)
rng = np.random.default_rng(7)
zipf = base.subset(np.arange(base.n))
perm = rng.permutation(np.arange(3, dims.vocab)).astype(np.int32)
r = np.minimum(rng.zipf(1.1, size=zipf.ids.size) - 1, perm.size - 1)
zipf.ids[:] = perm[r]
freq, lex = synth.shortlist_tables(dims.vocab, 100, 100, seed=85)
dev = torch.device("cuda:0")
st = torch.cuda.current_stream()
flush = torch.empty(128 << 20, dtype=torch.float32, device=dev)


def run(ss, sl):
    ids = torch.from_numpy(ss.ids).to(dev)
    cap = int(ss.max_len.sum())
    out = torch.zeros(cap, dtype=torch.int32, device=dev)
    ln = torch.zeros(ss.n, dtype=torch.int32, device=dev)
    f = lambda: m.translate_device(ids.data_ptr(), ss.offsets, ss.max_len, budget, out.data_ptr(),
                                   cap, ln.data_ptr(), st, shortlist=sl)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    ms = []
    for _ in range(5):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        f()
        b.record(st)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    return statistics.median(ms), int(ln.sum())


def union_sizes(ss):
    import oracle.oracle as O   # sizes only (reported context), not on the timed path
    order, off = O.batch_by_words(ss.lengths, budget)
    return [O.build_shortlist(dims.vocab, freq, lex, ss.subset(order[off[b]:off[b + 1]]).ids).size
            for b in range(len(off) - 1)]


for name, ss, tabs in [("plain", base, None), ("sl-full", base, (np.arange(dims.vocab), lex[:, :0])),
                       ("sl-unif", base, (freq, lex)), ("plain-zipf", zipf, None),
                       ("sl-zipf", zipf, (freq, lex))]:
    if tabs is not None:
        m.set_shortlist(*tabs)
    ms, words = run(ss, tabs is not None)
    rec = {"variant": name, "ms_per_job": ms, "words": words, "words_per_s": words / ms * 1e3}
    if tabs is not None and name != "sl-full":
        sz = union_sizes(ss)
        rec["batch_shortlist_mean"] = float(np.mean(sz))
        rec["batch_shortlist_max"] = int(max(sz))
    print(json.dumps(rec), flush=True)
