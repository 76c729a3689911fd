"""Job time vs number of decoder steps (max_len capped): separates encoder and per-step cost."""
import os, sys, json
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_1805_12096_b200 import mnmt as M

preset = sys.argv[1] if len(sys.argv) > 1 else "small-aan"
dims = synth.PRESETS[preset]
w = synth.make_weights(dims, seed=1)
m = M.Model(dims, w)
ss = synth.newstest_set()
dev = torch.device("cuda:0")
ids = torch.from_numpy(ss.ids).to(dev)
cap = int(ss.max_len.sum())
out = torch.zeros(cap, dtype=torch.int32, device=dev)
ln = torch.zeros(ss.n, dtype=torch.int32, device=dev)
st = torch.cuda.current_stream()
for lanes in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,4").split(",")]:
    m.set_option("lanes", lanes)
    m.set_option("max_concurrent_rows", 4096)
    for cap_steps in (1, 2, 10, 25, 50, 200):
        ml = np.minimum(ss.max_len, cap_steps).astype(np.int32)
        for _ in range(2):
            m.translate_device(ids.data_ptr(), ss.offsets, ml, 8192, out.data_ptr(), cap, ln.data_ptr(), st)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(st)
        for _ in range(3):
            m.translate_device(ids.data_ptr(), ss.offsets, ml, 8192, out.data_ptr(), cap, ln.data_ptr(), st)
        e.record(st); e.synchronize()
        stt = m.stats()
        print(f"lanes={lanes} steps<={cap_steps:4d}: {s.elapsed_time(e)/3:8.2f} ms  decode_steps={stt['decode_steps']} launches={stt['gpu_launches']}", flush=True)

# per-phase-type breakdown of the persistent step kernel (lane 0, one wave)
m.set_option("lanes", 1)
m.set_option("megakernel", 1)
m.set_option("profile_phases", 1)
for cap_steps in (1, 200):
    ml = np.minimum(ss.max_len, cap_steps).astype(np.int32)
    m.translate_device(ids.data_ptr(), ss.offsets, ml, 8192, out.data_ptr(), cap, ln.data_ptr(), st)
    torch.cuda.synchronize()
    prof, steps = m.phase_profile()
    tot = sum(prof.values())
    print(f"steps={steps} total={tot/1e6:.2f} ms per-step={tot/max(steps,1)/1e3:.1f} us",
          {k: f"{v/max(steps,1)/1e3:.1f}us" for k, v in prof.items()})
