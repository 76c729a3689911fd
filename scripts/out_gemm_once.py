"""One output-layer GEMM+argmax launch at the configs[1] early-step shape (for ncu)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_12096_b200 import mnmt as M
Mr, N, K = int(os.environ.get("M", 3072)), 36000, 256
dev = torch.device("cuda:0")
A = torch.randint(-127, 128, (Mr, K), dtype=torch.int8, device=dev)
W = torch.randint(-127, 128, (N, K), dtype=torch.int8, device=dev)
b = torch.zeros(N, device=dev)
keys = torch.zeros(Mr, dtype=torch.int64, device=dev)
for _ in range(3):
    M.op_gemm_i8(A.data_ptr(), W.data_ptr(), Mr, N, K, b.data_ptr(), 2.0, M.EPI_ARGMAX, keys.data_ptr(), None, 0, None)
torch.cuda.synchronize()
