"""Where the tiered-lane job's time goes (newstest job, bench options): the whole job, the critical
tier (longest sentences, last lane) alone, and the other tiers alone.
env PRESET, LANES, TIERS, GREEN, OPTS="smallm=32,sab=32,..." (extra model options)"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_1805_12096_b200 import mnmt as M
dims = synth.PRESETS[os.environ.get("PRESET", "small-aan")]
m = M.Model(dims, synth.make_weights(dims, 1))
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
ss = synth.newstest_set(seed=2014)
G, TIERS = int(os.environ.get("GREEN", 48)), int(os.environ.get("TIERS", 40))
LANES = int(os.environ.get("LANES", 3))
EXTRA = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in filter(None, os.environ.get("OPTS", "").split(","))}


def t_job(sub, opts, reps=5):
    for k, v in opts.items():
        m.set_option(k, v)
    ids = torch.from_numpy(sub.ids).to(dev)
    cap = int(sub.max_len.sum())
    out = torch.zeros(cap, dtype=torch.int32, device=dev); ln = torch.zeros(sub.n, dtype=torch.int32, device=dev)
    f = lambda: m.translate_device(ids.data_ptr(), sub.offsets, sub.max_len, 8192, out.data_ptr(), cap, ln.data_ptr(), st)
    f(); f(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(st); f(); b.record(st); b.synchronize(); ts.append(a.elapsed_time(b))
    return float(np.median(ts))


bench = dict(max_concurrent_rows=4096, lanes=LANES, lane_tiers=TIERS, green_sms=G, pers_reserve=16, **EXTRA)
print(f"whole job, bench options: {t_job(ss, bench):.2f} ms", flush=True)
# the tier split of mnmt_translate: contiguous length order, equal shares of sum S^p
order = np.argsort(ss.lengths, kind="stable")
w = ss.lengths[order].astype(np.float64) ** (TIERS / 10.0)
cut = int(np.searchsorted(np.cumsum(w), w.sum() * (LANES - 1) / LANES))
crit, bulk = order[cut + 1:], order[:cut + 1]
print(f"critical tier: {len(crit)} sentences, lengths {ss.lengths[crit].min()}..{ss.lengths[crit].max()}")
one = dict(max_concurrent_rows=4096, lanes=1, lane_tiers=0, green_sms=0, pers_reserve=0, **EXTRA)
print(f"critical tier alone, whole GPU: {t_job(ss.subset(crit), one):.2f} ms", flush=True)
two = dict(max_concurrent_rows=4096, lanes=max(1, LANES - 1), lane_tiers=TIERS, green_sms=0, pers_reserve=0, **EXTRA)
print(f"other tiers alone ({max(1, LANES - 1)} lanes), whole GPU: {t_job(ss.subset(bulk), two):.2f} ms", flush=True)
