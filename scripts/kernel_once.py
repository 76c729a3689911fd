"""One launch (after warm-up) of a decoder kernel at the bench shape, for ncu.
usage: KERNEL=dxd|out|topk|attn|attn16 M=630 python scripts/kernel_once.py"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_12096_b200 import mnmt as M
k = os.environ.get("KERNEL", "dxd")
Mr = int(os.environ.get("M", 630))
d, V, H = 256, 36000, 8
dev = torch.device("cuda:0")
if k == "topk":   # beam-search output GEMM (EPI_TOPK partials)
    A = torch.randint(-127, 128, (Mr, d), dtype=torch.int8, device=dev)
    W = torch.randint(-127, 128, (V, d), dtype=torch.int8, device=dev)
    b = torch.zeros(V, device=dev)
    out = torch.empty(Mr * 2 * ((V + 255) // 256) * M.TOPK_RECORD_BYTES, dtype=torch.uint8, device=dev)
    for _ in range(4):
        M.op_gemm_i8(A.data_ptr(), W.data_ptr(), Mr, V, d, b.data_ptr(), 2.0, M.EPI_TOPK, out.data_ptr(), None, int(os.environ.get("TOPK", 8)), None)
elif k in ("dxd", "out"):
    N = d if k == "dxd" else V
    A = torch.randint(-127, 128, (Mr, d), dtype=torch.int8, device=dev)
    W = torch.randint(-127, 128, (N, d), dtype=torch.int8, device=dev)
    b = torch.zeros(N, device=dev)
    out = torch.empty((Mr, N) if k == "dxd" else (Mr,), dtype=torch.float32 if k == "dxd" else torch.int64, device=dev)
    epi = M.EPI_F32 if k == "dxd" else M.EPI_ARGMAX
    for _ in range(4):
        M.op_gemm_i8(A.data_ptr(), W.data_ptr(), Mr, N, d, b.data_ptr(), 2.0, epi, out.data_ptr(), None,
                     int(os.environ.get("NTILE", 0)), None)   # NTILE=-1: the small-M kernel
else:
    S = int(os.environ.get("S", 21))
    L = np.full(Mr, S, np.int32); st = (np.arange(Mr) * S).astype(np.int32)
    kv = torch.randn(Mr * S, 2 * d, device=dev); q = torch.randn(Mr, d, device=dev)
    if k == "attn16":   # bf16 source K/V (F3)
        kv = kv.to(torch.bfloat16)
    op = M.op_attention_bf16 if k == "attn16" else M.op_attention
    S, Ln = torch.from_numpy(st).to(dev), torch.from_numpy(L).to(dev)
    oq = torch.empty(Mr, d, dtype=torch.int8, device=dev)
    for _ in range(4):
        op(q.data_ptr(), d, kv.data_ptr(), 2 * d, 0, d, S.data_ptr(), Ln.data_ptr(), Mr, d, H, 2.0, oq.data_ptr(), None, None)
torch.cuda.synchronize()
