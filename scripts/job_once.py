"""One full translation job (after 2 warm-up jobs) inside an NVTX range "job", for an ncu
launch list of exactly one job:  ncu --nvtx --nvtx-include "job/" ... python scripts/job_once.py
(env PRESET, MCR, BEAM, OPTS = bench launch options)"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_1805_12096_b200 import mnmt as M
dims = synth.PRESETS[os.environ.get("PRESET", "small-aan")]
m = M.Model(dims, synth.make_weights(dims, 1))
m.set_option("max_concurrent_rows", int(os.environ.get("MCR", 4096)))
# bench.py's launch options for the workload (env OPTS="lanes=3,lane_tiers=40,..."); the default
# omits green_sms: kernels in a green context are not profiled by ncu
for kv in filter(None, os.environ.get("OPTS", "lanes=3,lane_tiers=40,pers_reserve=16").split(",")):
    k, v = kv.split("=")
    m.set_option(k, int(v))
ss = synth.newstest_set(seed=2014)
if os.environ.get("LMAX") or os.environ.get("LMIN"):   # a length slice (bulk tiers: LMAX=45)
    keep = [i for i in range(ss.n) if int(os.environ.get("LMIN", 0)) <= ss.lengths[i] <= int(os.environ.get("LMAX", 1 << 30))]
    ss = ss.subset(keep)
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
ids = torch.from_numpy(ss.ids).to(dev)
cap = int(ss.max_len.sum())
out = torch.zeros(cap, dtype=torch.int32, device=dev); ln = torch.zeros(ss.n, dtype=torch.int32, device=dev)
beam = int(os.environ.get("BEAM", 0))   # > 0: beam search job (mnmt_beam_translate)
if beam:
    out = torch.zeros(cap * beam, dtype=torch.int32, device=dev)
    ln = torch.zeros(ss.n * beam, dtype=torch.int32, device=dev)
    sc = torch.zeros(ss.n * beam, dtype=torch.float32, device=dev)
    nh = torch.zeros(ss.n, dtype=torch.int32, device=dev)
    f = lambda: m.beam_translate_device(ids.data_ptr(), ss.offsets, ss.max_len, 8192, beam, out.data_ptr(),
                                        cap * beam, ln.data_ptr(), sc.data_ptr(), nh.data_ptr(), st)
else:
    f = lambda: m.translate_device(ids.data_ptr(), ss.offsets, ss.max_len, 8192, out.data_ptr(), cap, ln.data_ptr(), st)
f(); f(); torch.cuda.synchronize()
torch.cuda.nvtx.range_push("job"); f(); torch.cuda.nvtx.range_pop(); torch.cuda.synchronize()
s = m.stats(); print("launches", s["gpu_launches"], "steps", s["decode_steps"], "words", int(ln.sum()))
