"""Decoder source attention alone (op-level ABI, CUDA graph of 100 launches): us per launch."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_12096_b200 import mnmt as M
dev = torch.device("cuda:0"); d, H = 256, 8
def t(fn, iters=100):
    for _ in range(3): fn(torch.cuda.current_stream())
    torch.cuda.synchronize(); g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(iters): fn(torch.cuda.current_stream())
    g.replay(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record(); g.replay(); b.record(); b.synchronize(); return 1000 * a.elapsed_time(b) / iters
for rows, S in ((630, 21), (128, 60), (64, 90), (2048, 15)):
    L = np.full(rows, S, np.int32); st = (np.arange(rows) * S).astype(np.int32)
    # K/V of several layers' worth so it does not sit in L2 between launches
    kv = torch.randn(rows * S * 8, 2 * d, device=dev); q = torch.randn(rows, d, device=dev)
    Sd, Ld = torch.from_numpy(st).to(dev), torch.from_numpy(L).to(dev)
    oq = torch.empty(rows, d, dtype=torch.int8, device=dev)
    us = t(lambda s_: M.op_attention(q.data_ptr(), d, kv.data_ptr(), 2 * d, 0, d, Sd.data_ptr(), Ld.data_ptr(), rows, d, H, 2.0, oq.data_ptr(), None, s_))
    print(f"rows {rows} S {S}: {us:.2f} us", flush=True)
