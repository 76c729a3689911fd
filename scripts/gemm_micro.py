"""Warm in-chain latency of the decoder GEMMs: 200 launches captured in a CUDA graph (PDL chain),
average per launch, at the big / base widths.  usage: python scripts/gemm_micro.py [D F]
(env SMALLM=1: rows <= 32 take the small-M IDP4A kernel, n_tile -1)"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_12096_b200 import mnmt as M
import bench
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
d = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
F = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
for name, N, K, epi in (("dxd", d, d, M.EPI_F32), ("qkv", 3 * d, d, M.EPI_F32), ("ffn1", F, d, M.EPI_RELU_Q),
                        ("ffn2", d, F, M.EPI_F32)):
    for m in (8, 32, 128, 256, 630):
        A = torch.randint(-127, 128, (m, K), dtype=torch.int8, device=dev)
        W = torch.randint(-127, 128, (N, K), dtype=torch.int8, device=dev)
        b = torch.zeros(N, device=dev)
        out = torch.empty((m, N), dtype=torch.int8 if epi == M.EPI_RELU_Q else torch.float32, device=dev)
        nt = -1 if (os.environ.get("SMALLM") == "1" and m <= 32) else 0
        fn = lambda s: M.op_gemm_i8(A.data_ptr(), W.data_ptr(), m, N, K, b.data_ptr(), 2.0, epi, out.data_ptr(), None, nt, s)
        ms = bench.time_kernel(fn, 200, st)
        print(f"{name} M={m:4d} N={N:5d} K={K:5d}: {1000 * ms:7.2f} us  {2.0 * m * N * K / (ms * 1e-3) / 1e12:7.1f} TOP/s", flush=True)
