"""Warm in-chain latency of the row kernels: 200 launches of one op captured in a CUDA graph
(PDL chain), average per launch.  usage: python scripts/row_micro.py [ln|attn] (env as the lib)"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_12096_b200 import mnmt as M
import bench
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
what = sys.argv[1] if len(sys.argv) > 1 else "ln"
for d in (256, 512, 1024):
    for n in (32, 128, 256, 630, 2048):
        if what == "ln":
            x = torch.randn(n, d, device=dev); dl = torch.randn(n, d, device=dev)
            g = torch.ones(d, device=dev); b = torch.zeros(d, device=dev)
            out = torch.empty(n, d, device=dev); oq = torch.empty(n, d, dtype=torch.int8, device=dev)
            fn = lambda s: M.op_layernorm(x.data_ptr(), dl.data_ptr(), None, None, g.data_ptr(), b.data_ptr(), n, d, 1e-6, 2.0, out.data_ptr(), oq.data_ptr(), s)
            byt = 13.0 * n * d
        else:
            H = 16 if d == 1024 else 8
            S = 21
            L = np.full(n, S, np.int32); sst = (np.arange(n) * S).astype(np.int32)
            kv = torch.randn(n * S, 2 * d, device=dev); q = torch.randn(n, d, device=dev)
            Sd, Ld = torch.from_numpy(sst).to(dev), torch.from_numpy(L).to(dev)
            oq = torch.empty(n, d, dtype=torch.int8, device=dev)
            if what == "src":   # the decode path's kernel choice (TMA tiles)
                fn = lambda s: M.op_src_attention(q.data_ptr(), d, kv.data_ptr(), n * S, 2 * d, 0, d, Sd.data_ptr(), Ld.data_ptr(), S, n, d, H, 2.0, oq.data_ptr(), None, s)
            else:
                fn = lambda s: M.op_attention(q.data_ptr(), d, kv.data_ptr(), 2 * d, 0, d, Sd.data_ptr(), Ld.data_ptr(), n, d, H, 2.0, oq.data_ptr(), None, s)
            byt = 8.0 * n * S * d
        ms = bench.time_kernel(fn, 200, st)
        print(f"{what} d={d:5d} rows={n:5d}: {1000 * ms:8.2f} us/launch  {byt / (ms * 1e-3) / 1e9:8.1f} GB/s (warm)", flush=True)
