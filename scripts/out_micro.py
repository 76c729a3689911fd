"""Output GEMM + argmax (N = 36,000) at few rows: the one-shot kernel vs the persistent one
(MNMT_GEMM_PERSISTENT decides per process), per launch in a PDL chain of 100, twice."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_12096_b200 import mnmt as M
import bench
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
d = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
N = 36000
W = torch.randint(-127, 128, (N, d), dtype=torch.int8, device=dev)
b = torch.zeros(N, device=dev)
for m in (1, 2, 8, 16, 32, 48, 64, 96, 128):
    A = torch.randint(-127, 128, (m, d), dtype=torch.int8, device=dev)
    out = torch.zeros(m, dtype=torch.int64, device=dev)
    res = []
    for nt in (0, 128, 256):
        fn = lambda s: M.op_gemm_i8(A.data_ptr(), W.data_ptr(), m, N, d, b.data_ptr(), 2.0, M.EPI_ARGMAX, out.data_ptr(), None, nt, s)
        t1 = bench.time_kernel(fn, 100, st); t2 = bench.time_kernel(fn, 100, st)
        res.append(f"bn{nt} {1000 * t1:6.2f}/{1000 * t2:6.2f}")
    print(f"d {d} M={m:4d}: " + " | ".join(res), flush=True)
