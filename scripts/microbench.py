"""Per-launch device time of individual libmnmt kernels inside a CUDA graph (back-to-back,
PDL-enabled launches), through the op-level C-ABI.  Run on the GPU box."""
import sys, os, json
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_12096_b200 import mnmt as M

dev = torch.device("cuda:0")
torch.cuda.set_device(0)


def graph_time(fn, iters=50):
    for _ in range(3):
        fn(torch.cuda.current_stream())
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        cs = torch.cuda.current_stream()
        for _ in range(iters):
            fn(cs)
    g.replay(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); g.replay(); e.record(); e.synchronize()
    return 1000 * s.elapsed_time(e) / iters   # us


def codes(shape):
    return torch.randint(-127, 128, shape, dtype=torch.int8, device=dev)


res = {}
for (Mr, N, K, epi, name) in [(3072, 256, 256, M.EPI_F32, "dxd f32 M3072"), (384, 256, 256, M.EPI_F32, "dxd f32 M384"),
                              (128, 256, 256, M.EPI_F32, "dxd f32 M128"),
                              (3072, 2048, 256, M.EPI_RELU_Q, "ffn1 M3072"), (3072, 256, 2048, M.EPI_F32, "ffn2 M3072"),
                              (3072, 36000, 256, M.EPI_ARGMAX, "out M3072"), (384, 36000, 256, M.EPI_ARGMAX, "out M384"),
                              (62954, 768, 256, M.EPI_F32, "enc qkv M63k"), (62954, 3072, 256, M.EPI_F32, "enc kv M63k")]:
    A, W = codes((Mr, K)), codes((N, K))
    b = torch.zeros(N, device=dev)
    out = torch.empty((Mr, N) if epi != M.EPI_ARGMAX else (Mr,), dtype=torch.float32 if epi in (M.EPI_F32,) else (torch.int8 if epi == M.EPI_RELU_Q else torch.int64), device=dev)
    for bn in (0, 64, 128, 256):
        t = graph_time(lambda st: M.op_gemm_i8(A.data_ptr(), W.data_ptr(), Mr, N, K, b.data_ptr(), 2.0, epi, out.data_ptr(), None, bn, st), 20)
        ops = 2.0 * Mr * N * K
        res[f"gemm {name} bn{bn}"] = (round(t, 2), round(ops / t / 1e6, 1))
for n in (384, 3072):
    d = 256
    x, y, g_, b_ = (torch.randn(n, d, device=dev), torch.randn(n, d, device=dev), torch.ones(d, device=dev), torch.zeros(d, device=dev))
    o, oq = torch.empty(n, d, device=dev), torch.empty(n, d, dtype=torch.int8, device=dev)
    res[f"ln n{n}"] = round(graph_time(lambda st: M.op_layernorm(x.data_ptr(), y.data_ptr(), None, None, g_.data_ptr(), b_.data_ptr(), n, d, 1e-6, 2.0, o.data_ptr(), oq.data_ptr(), st)), 2)
    res[f"gate-ln n{n}"] = round(graph_time(lambda st: M.op_layernorm(x.data_ptr(), y.data_ptr(), x.data_ptr(), y.data_ptr(), g_.data_ptr(), b_.data_ptr(), n, d, 1e-6, 2.0, o.data_ptr(), oq.data_ptr(), st)), 2)
    L = np.full(n, 21, np.int32); st_ = np.arange(n, dtype=np.int32) * 21
    kv = torch.randn(n * 21, 2 * d, device=dev); q = torch.randn(n, d, device=dev)
    S, Ln = torch.from_numpy(st_).to(dev), torch.from_numpy(L).to(dev)
    oq2 = torch.empty(n, d, dtype=torch.int8, device=dev)
    res[f"attn n{n} S21"] = round(graph_time(lambda st: M.op_attention(q.data_ptr(), d, kv.data_ptr(), 2 * d, 0, d, S.data_ptr(), Ln.data_ptr(), n, d, 8, 2.0, oq2.data_ptr(), None, st)), 2)
    qq = torch.empty(n * d, dtype=torch.int8, device=dev)
    res[f"quantize n{n}xd"] = round(graph_time(lambda st: M.op_quantize(x.data_ptr(), n * d, 2.0, qq.data_ptr(), st)), 2)
for k, v in res.items():
    print(f"{k:32s} {v}")
