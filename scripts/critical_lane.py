"""Job time of the longest length tier alone (the critical path of the tiered-lane schedule)
vs the whole newstest job, same options (lanes/tiers/priorities)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_1805_12096_b200 import mnmt as M
dims = synth.PRESETS["small-aan"]
m = M.Model(dims, synth.make_weights(dims, 1))
m.set_option("max_concurrent_rows", 4096)
for k, v in (a.split("=") for a in sys.argv[1:]):
    m.set_option(k, int(v))
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
ss = synth.newstest_set(seed=2014)
order = np.argsort(ss.lengths, kind="stable")


def t_job(sub, lanes, tiers, reps=5):
    m.set_option("lanes", lanes); m.set_option("lane_tiers", tiers)
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


print(f"whole job, 3 lanes tiers 30: {t_job(ss, 3, 30):.2f} ms")
for k in (100, 206, 400):
    sub = ss.subset(order[-k:])
    print(f"longest {k} sentences alone (1 lane): {t_job(sub, 1, 0):.2f} ms")
sub = ss.subset(order[:-206])
print(f"all but the longest 206 (2 lanes tiers 30): {t_job(sub, 2, 30):.2f} ms")
for k in (206,):
    sub = ss.subset(order[-k:])
    cap1 = synth.SentenceSet(sub.ids, sub.offsets, np.minimum(sub.max_len, 1).astype(np.int32))
    print(f"longest {k} sentences, 1 decoder step (encoder + 1 step): {t_job(cap1, 1, 0):.2f} ms")
