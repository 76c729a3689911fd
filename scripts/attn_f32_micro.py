"""Source attention through the decode path's TMA kernel, per launch (4 K/V copies rotated so the
K/V stream is HBM-cold), at the big student's shapes; run with and without MNMT_ATTN_F32=1."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_12096_b200 import mnmt as M
dev = torch.device("cuda:0")
d, H = 1024, 16


def t(fn, iters=40):
    for i in range(4): fn(torch.cuda.current_stream(), i)
    torch.cuda.synchronize(); g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(iters): fn(torch.cuda.current_stream(), i)
    g.replay(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record(); g.replay(); b.record(); b.synchronize(); return 1000 * a.elapsed_time(b) / iters


for rows, S in ((630, 21), (2048, 15), (632, 48), (128, 60), (630, 12), (2048, 8), (256, 16), (32, 80)):
    L = np.full(rows, S, np.int32); st = (np.arange(rows) * S).astype(np.int32)
    copies = max(1, min(8, int(np.ceil(160e6 / (rows * S * 8 * d)))))
    kvs = [torch.randn(rows * S, 2 * d, device=dev) for _ in range(copies)]
    q = torch.randn(rows, d, device=dev)
    Sd, Ld = torch.from_numpy(st).to(dev), torch.from_numpy(L).to(dev)
    oq = torch.empty(rows, d, dtype=torch.int8, device=dev)
    us = t(lambda s_, i: M.op_src_attention(q.data_ptr(), d, kvs[i % copies].data_ptr(), rows * S, 2 * d, 0, d,
                                            Sd.data_ptr(), Ld.data_ptr(), S, rows, d, H, 2.0, oq.data_ptr(), None, s_))
    gbs = rows * S * 2 * d * 4 / (us * 1e-6) / 1e9
    print(f"{'fp32' if os.environ.get('MNMT_ATTN_F32') == '1' else 'fp64'} warps={os.environ.get('MNMT_AT_WARPS', '4')} rows {rows:5d} S {S:3d}: {us:7.2f} us ({gbs:6.0f} GB/s)", flush=True)
