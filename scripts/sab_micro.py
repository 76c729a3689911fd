"""Warm in-chain latency (200 launches in a PDL graph) of the decoder GEMMs at small row counts:
the 128-row tcgen05 kernel (n_tile 0), the small-M IDP4A kernel (-1, <= 32 rows) and the swap-AB
tcgen05 kernel (-2) at several split-K caps.  usage: python scripts/sab_micro.py [D F]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_12096_b200 import mnmt as M
import bench
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
d = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
F = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
V = 36000
rows = [int(x) for x in os.environ.get("ROWS", "1,8,16,32,64,128").split(",")]
for name, N, K, epi in (("dxd", d, d, M.EPI_F32), ("qkv", 3 * d, d, M.EPI_F32), ("ffn1", F, d, M.EPI_RELU_Q),
                        ("ffn2", d, F, M.EPI_F32), ("out", V, d, M.EPI_ARGMAX)):
    for m in rows:
        A = torch.randint(-127, 128, (m, K), dtype=torch.int8, device=dev)
        W = torch.randint(-127, 128, (N, K), dtype=torch.int8, device=dev)
        b = torch.zeros(N, device=dev)
        if epi == M.EPI_ARGMAX:
            out = torch.zeros(m, dtype=torch.int64, device=dev)
        else:
            out = torch.empty((m, N), dtype=torch.int8 if epi == M.EPI_RELU_Q else torch.float32, device=dev)
        res = []
        variants = [("tc128", 0, -1)]
        if m <= 32 and epi != M.EPI_ARGMAX:
            variants.append(("idp4a", -1, 1))
        kb = K // 128
        for ks in (1, 2, 4, 8):
            if ks == 1 or kb >= 2 * ks:
                variants.append((f"sab/ks{ks}", -2, ks))
        for vn, nt, ks in variants:
            if nt == -1:
                fn = lambda s: M.op_gemm_i8(A.data_ptr(), W.data_ptr(), m, N, K, b.data_ptr(), 2.0, epi,
                                            out.data_ptr(), None, nt, s)
            else:
                fn = lambda s: M.op_gemm_i8_split(A.data_ptr(), W.data_ptr(), m, N, K, b.data_ptr(), 2.0, epi,
                                                  out.data_ptr(), None, nt, ks if nt == -2 else 1, s)
            try:
                ms = bench.time_kernel(fn, 200, st)
                res.append(f"{vn} {1000 * ms:6.2f}")
            except Exception as e:   # noqa: BLE001
                res.append(f"{vn} err({str(e)[:40]})")
        print(f"{name:4s} M={m:4d} N={N:5d} K={K:5d}: " + " | ".join(res), flush=True)
