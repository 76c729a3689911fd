"""Time the whole job vs the job capped at 1 decoder step (~ encoder + 1 step), device-resident.
Under ncu with ENC_ONLY=1 the capped job runs once after warm-up (launch list of the encoder)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_1805_12096_b200 import mnmt as M
preset = os.environ.get("PRESET", "small-aan")
dims = synth.PRESETS[preset]
m = M.Model(dims, synth.make_weights(dims, 1))
m.set_option("max_concurrent_rows", 4096)
ss = synth.newstest_set(seed=2014)
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
ids = torch.from_numpy(ss.ids).to(dev)
def run(cap, reps):
    ml = np.minimum(ss.max_len, cap).astype(np.int32)
    out = torch.zeros(int(ml.sum()), dtype=torch.int32, device=dev)
    ln = torch.zeros(ss.n, dtype=torch.int32, device=dev)
    f = lambda: m.translate_device(ids.data_ptr(), ss.offsets, ml, 8192, out.data_ptr(), int(ml.sum()), ln.data_ptr(), st)
    for _ in range(2): f()
    torch.cuda.synchronize()
    if os.environ.get("ENC_ONLY"):
        torch.cuda.nvtx.range_push("job"); f(); torch.cuda.nvtx.range_pop(); torch.cuda.synchronize(); return 0
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(st); f(); b.record(st); b.synchronize(); ts.append(a.elapsed_time(b))
    return float(np.median(ts))
if os.environ.get("ENC_ONLY"):
    run(1, 1)
else:
    for cap in (1, 2, 200):
        print(f"{preset} max_len cap {cap}: {run(cap, 5):.2f} ms", flush=True)
