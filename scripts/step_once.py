"""One decode of B sentences of length T (after a warm-up), inside an NVTX range "job", for an
ncu launch list of the per-step kernels at a fixed row count (env B, T, PRESET)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_1805_12096_b200 import mnmt as M
dims = synth.PRESETS[os.environ.get("PRESET", "small-aan")]
B, T = int(os.environ.get("B", 2048)), int(os.environ.get("T", 8))
m = M.Model(dims, synth.make_weights(dims, 1))
ss = synth.uniform_set(B, T, seed=5)
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
ids = torch.from_numpy(ss.ids).to(dev)
out = torch.zeros(B * T, dtype=torch.int32, device=dev); ln = torch.zeros(B, dtype=torch.int32, device=dev)
f = lambda: m.translate_device(ids.data_ptr(), ss.offsets, ss.max_len, 1 << 30, out.data_ptr(), B * T, ln.data_ptr(), st)
f(); torch.cuda.synchronize()
torch.cuda.nvtx.range_push("job"); f(); torch.cuda.nvtx.range_pop(); torch.cuda.synchronize()
print("steps", m.stats()["decode_steps"])
