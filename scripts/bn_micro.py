"""Decoder GEMMs at 128-640 rows: the N tile picked by the library (0) vs forced 64 / 128 / 256, per
launch in a PDL chain of 200 (big student widths)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_12096_b200 import mnmt as M
import bench
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
for name, N, K, epi in (("dxd", 1024, 1024, M.EPI_F32), ("qkv", 3072, 1024, M.EPI_F32), ("ffn1", 4096, 1024, M.EPI_RELU_Q),
                        ("ffn2", 1024, 4096, M.EPI_F32)):
    for m in (128, 256, 384, 630):
        A = torch.randint(-127, 128, (m, K), dtype=torch.int8, device=dev)
        W = torch.randint(-127, 128, (N, K), dtype=torch.int8, device=dev)
        b = torch.zeros(N, device=dev)
        out = torch.empty((m, N), dtype=torch.int8 if epi == M.EPI_RELU_Q else torch.float32, device=dev)
        res = []
        for nt in (0, 64, 128, 256):
            fn = lambda s: M.op_gemm_i8(A.data_ptr(), W.data_ptr(), m, N, K, b.data_ptr(), 2.0, epi, out.data_ptr(), None, nt, s)
            res.append(f"bn{nt} {1000 * bench.time_kernel(fn, 200, st):6.2f}")
        for ks in (2, 4):
            fn = lambda s: M.op_gemm_i8_split(A.data_ptr(), W.data_ptr(), m, N, K, b.data_ptr(), 2.0, epi, out.data_ptr(), None, 0, ks, s)
            res.append(f"ks{ks} {1000 * bench.time_kernel(fn, 200, st):6.2f}")
        print(f"{name:4s} M={m:4d} N={N:5d} K={K:5d}: " + " | ".join(res), flush=True)
