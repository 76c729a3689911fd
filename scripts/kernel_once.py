"""One launch (after warm-up) of a decoder kernel at a bench shape, for ncu.
usage: KERNEL=dxd|ffn1|ffn2|out|topk|attn|attn16|ln|enc M=630 D=256 F=2048 H=8 S=21 python scripts/kernel_once.py
(NTILE=-1: the small-M GEMM kernel; NTILE=64/128/256: a fixed tcgen05 N tile)"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_12096_b200 import mnmt as M
k = os.environ.get("KERNEL", "dxd")
Mr = int(os.environ.get("M", 630))
d, V, H = int(os.environ.get("D", 256)), 36000, int(os.environ.get("H", 8))
F = int(os.environ.get("F", 2048))
dev = torch.device("cuda:0")
if k == "topk":   # beam-search output GEMM (EPI_TOPK partials)
    A = torch.randint(-127, 128, (Mr, d), dtype=torch.int8, device=dev)
    W = torch.randint(-127, 128, (V, d), dtype=torch.int8, device=dev)
    b = torch.zeros(V, device=dev)
    out = torch.empty(Mr * 2 * ((V + 255) // 256) * M.TOPK_RECORD_BYTES, dtype=torch.uint8, device=dev)
    for _ in range(4):
        M.op_gemm_i8(A.data_ptr(), W.data_ptr(), Mr, V, d, b.data_ptr(), 2.0, M.EPI_TOPK, out.data_ptr(), None, int(os.environ.get("TOPK", 8)), None)
elif k in ("dxd", "out", "ffn1", "ffn2"):
    N, K = {"dxd": (d, d), "out": (V, d), "ffn1": (F, d), "ffn2": (d, F)}[k]
    A = torch.randint(-127, 128, (Mr, K), dtype=torch.int8, device=dev)
    W = torch.randint(-127, 128, (N, K), dtype=torch.int8, device=dev)
    b = torch.zeros(N, device=dev)
    if k == "out":
        out, out2, epi = torch.empty(Mr, dtype=torch.int64, device=dev), None, M.EPI_ARGMAX
    elif k == "ffn1":
        out, out2, epi = torch.empty((Mr, N), dtype=torch.int8, device=dev), None, M.EPI_RELU_Q
    else:
        out, out2, epi = torch.empty((Mr, N), dtype=torch.float32, device=dev), None, M.EPI_F32
    for _ in range(4):
        if k == "out":
            out.zero_()
        M.op_gemm_i8(A.data_ptr(), W.data_ptr(), Mr, N, K, b.data_ptr(), 2.0, epi, out.data_ptr(), None,
                     int(os.environ.get("NTILE", 0)), None)
elif k == "enc":   # encoder self-attention: M sentences of 1..S tokens (env ENCV = op variant)
    S = int(os.environ.get("S", 28))
    rng = np.random.default_rng(5)
    L = rng.integers(max(1, S // 3), S + 1, size=Mr).astype(np.int32); L[0] = S
    st = np.concatenate([[0], np.cumsum(L)[:-1]]).astype(np.int32)
    qkv = torch.randn(int(L.sum()), 3 * d, device=dev)
    Sd, Ln = torch.from_numpy(st).to(dev), torch.from_numpy(L).to(dev)
    oq = torch.empty(int(L.sum()), d, dtype=torch.int8, device=dev)
    for _ in range(4):
        M.op_attention_enc(qkv.data_ptr(), Sd.data_ptr(), Ln.data_ptr(), Mr, d, H, S, 2.0, oq.data_ptr(),
                           int(os.environ.get("ENCV", 0)), None)
elif k == "ln":
    x = torch.randn(Mr, d, device=dev); dl = torch.randn(Mr, d, device=dev)
    g = torch.ones(d, device=dev); bb = torch.zeros(d, device=dev)
    out = torch.empty(Mr, d, device=dev); oq = torch.empty(Mr, d, dtype=torch.int8, device=dev)
    for _ in range(4):
        M.op_layernorm(x.data_ptr(), dl.data_ptr(), None, None, g.data_ptr(), bb.data_ptr(), Mr, d,
                       1e-6, 2.0, out.data_ptr(), oq.data_ptr(), None)
else:
    S = int(os.environ.get("S", 21))
    L = np.full(Mr, S, np.int32); st = (np.arange(Mr) * S).astype(np.int32)
    kv = torch.randn(Mr * S, 2 * d, device=dev); q = torch.randn(Mr, d, device=dev)
    if k == "attn16":   # bf16 source K/V (F3)
        kv = kv.to(torch.bfloat16)
    Sd, Ln = torch.from_numpy(st).to(dev), torch.from_numpy(L).to(dev)
    oq = torch.empty(Mr, d, dtype=torch.int8, device=dev)
    for _ in range(4):
        if k == "attn16":
            M.op_attention_bf16(q.data_ptr(), d, kv.data_ptr(), 2 * d, 0, d, Sd.data_ptr(), Ln.data_ptr(), Mr, d, H, 2.0, oq.data_ptr(), None, None)
        else:   # the decode path's choice (TMA tiles for d_h = 32 / 64)
            M.op_src_attention(q.data_ptr(), d, kv.data_ptr(), Mr * S, 2 * d, 0, d, Sd.data_ptr(), Ln.data_ptr(), S, Mr, d, H, 2.0, oq.data_ptr(), None, None)
torch.cuda.synchronize()
