"""Per-step decoder latency vs live rows: B sentences of length T decoded for T steps, minus the
same job capped at 1 step (encoder + first step), divided by T - 1.  Device-resident inputs."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_1805_12096_b200 import mnmt as M
preset = os.environ.get("PRESET", "small-aan")
dims = synth.PRESETS[preset]
m = M.Model(dims, synth.make_weights(dims, 1))
for k, v in (a.split("=") for a in sys.argv[1:]):
    m.set_option(k, int(v))
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
T = int(os.environ.get("T", 64))


def run(ss, cap, reps=5):
    ml = np.minimum(ss.max_len, cap).astype(np.int32)
    ids = torch.from_numpy(ss.ids).to(dev)
    out = torch.zeros(int(ml.sum()), dtype=torch.int32, device=dev)
    ln = torch.zeros(ss.n, dtype=torch.int32, device=dev)
    f = lambda: m.translate_device(ids.data_ptr(), ss.offsets, ml, 1 << 30, out.data_ptr(), int(ml.sum()), ln.data_ptr(), st)
    f(); f(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(st); f(); b.record(st); b.synchronize(); ts.append(a.elapsed_time(b))
    return float(np.median(ts))


for B in [int(x) for x in os.environ.get("BS", "1,8,32,128,256,512,1024,2048").split(",")]:
    ss = synth.uniform_set(B, T, seed=5)
    full, one = run(ss, T), run(ss, 1)
    print(f"{preset} B={B:5d} T={T}: {1000 * (full - one) / (T - 1):7.1f} us/step  (job {full:.2f} ms, encoder+1 step {one:.2f} ms)", flush=True)
