"""BASELINE configs[4]: base-AAN throughput over word budget x sentence length (1 GPU).

Uniform-length synthetic sets of >= 62,954 source words (max_len = S).  Batches follow the
paper's rule (>= budget words) and are decoded one at a time (no co-scheduling), so
the budget is the batch size.  Prints one JSON line per cell."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_1805_12096_b200 import mnmt as M

preset = os.environ.get("PRESET", "base-aan")
dims = synth.PRESETS[preset]
m = M.Model(dims, synth.make_weights(dims, 1))
m.set_option("max_concurrent_rows", 0)
st = torch.cuda.current_stream()
dev = torch.device("cuda:0")
budgets = [int(x) for x in os.environ.get("BUDGETS", "384,1024,2048,4096,8192,16384,32768,65536").split(",")]
lengths = [int(x) for x in os.environ.get("LENGTHS", "5,10,20,40,70,100").split(",")]
for S in lengths:
    n = max(1, -(-62954 // S))
    ss = synth.uniform_set(n, S, seed=S)
    ids = torch.from_numpy(ss.ids).to(dev)
    cap = int(ss.max_len.sum())
    out = torch.zeros(cap, dtype=torch.int32, device=dev)
    ln = torch.zeros(ss.n, dtype=torch.int32, device=dev)
    for B in budgets:
        run = lambda: m.translate_device(ids.data_ptr(), ss.offsets, ss.max_len, B, out.data_ptr(), cap, ln.data_ptr(), st)
        run(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        e0.record(st)
        for _ in range(reps):
            run()
        e1.record(st); e1.synchronize()
        ms = e0.elapsed_time(e1) / reps
        words = int(ln.sum().item())
        stt = m.stats()
        print(json.dumps({"preset": preset, "S": S, "budget": B, "sentences": ss.n, "batches": stt["batches"],
                          "steps": stt["decode_steps"], "ms": round(ms, 3),
                          "target_words_per_s": round(words / (ms / 1e3))}), flush=True)
