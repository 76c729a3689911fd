"""Many-row GEMMs: the one-CTA persistent kernel (BN 256, n_tile 256) vs the CTA-pair kernel
(n_tile -3), per launch in a CUDA graph of 20 launches; TOP/s and fraction of the int8 peak."""
import os, sys, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_12096_b200 import mnmt as M
import bench
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
peak = 2 * bench.load_peaks()["bf16_tflops"]
for name, Mr, N, K, epi in (("enc-qkv big", 33000, 3072, 1024, M.EPI_F32), ("enc-ffn1 big", 33000, 4096, 1024, M.EPI_RELU_Q),
                            ("enc-ffn2 big", 33000, 1024, 4096, M.EPI_F32), ("out big", 630, 36000, 1024, M.EPI_ARGMAX),
                            ("out big 2k", 2048, 36000, 1024, M.EPI_ARGMAX), ("enc-qkv base", 33000, 1536, 512, M.EPI_F32),
                            ("kv big", 33000, 12288, 1024, M.EPI_F32)):
    A = torch.randint(-127, 128, (Mr, K), dtype=torch.int8, device=dev)
    W = torch.randint(-127, 128, (N, K), dtype=torch.int8, device=dev)
    b = torch.zeros(N, device=dev)
    if epi == M.EPI_ARGMAX:
        out = torch.zeros(Mr, dtype=torch.int64, device=dev)
    else:
        out = torch.empty((Mr, N), dtype=torch.int8 if epi == M.EPI_RELU_Q else torch.float32, device=dev)
    res = []
    for nt in (256, -3):
        fn = lambda s: M.op_gemm_i8(A.data_ptr(), W.data_ptr(), Mr, N, K, b.data_ptr(), 2.0, epi, out.data_ptr(), None, nt, s)
        ms = bench.time_kernel(fn, 20, st)
        tops = 2.0 * Mr * N * K / (ms * 1e-3) / 1e12
        res.append(f"{'pers' if nt == 256 else 'pair'} {1000 * ms:8.1f} us {tops:6.0f} TOP/s ({100 * tops / peak:4.1f} %)")
    print(f"{name:13s} M={Mr:5d} N={N:5d} K={K:5d}: " + " | ".join(res), flush=True)
