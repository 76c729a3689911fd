"""Timeline of one int8 GEMM inside a PDL chain (mnmt_debug_gemm_chain): where the ~3 us go."""
import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_12096_b200 import mnmt as M
L = M.lib()
L.mnmt_debug_gemm_chain.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p]
dev = torch.device("cuda:0")
SHAPES = ((8, 256, 256), (128, 256, 256), (630, 256, 256), (8, 2048, 256), (8, 256, 2048), (630, 2048, 256))
if os.environ.get("SHAPES"):   # e.g. SHAPES="8x1024x1024,128x1024x1024"
    SHAPES = tuple(tuple(int(v) for v in s.split("x")) for s in os.environ["SHAPES"].split(","))
for (Mr, N, K) in SHAPES:
    A = torch.randint(-127, 128, (max(Mr, 128), K), dtype=torch.int8, device=dev)
    W = torch.randint(-127, 128, (N, K), dtype=torch.int8, device=dev)
    out = torch.empty(Mr, N, device=dev)
    res = (C.c_double * 11)()
    st = L.mnmt_debug_gemm_chain(A.data_ptr(), W.data_ptr(), Mr, N, K, out.data_ptr(), 200, res)
    assert st == 0, M.lib().mnmt_last_error()
    print(f"M {Mr:4d} N {N:4d} K {K:4d}: {res[0]:.2f} us/launch | wait {res[1]:.2f} operands {res[2]:.2f} "
          f"acc {res[3]:.2f} tmem-ld {res[8]:.2f} dequant {res[9]:.2f} staged {res[10]:.2f} stores {res[4]:.2f} end {res[5]:.2f} | entry-to-entry {res[6]:.2f} | end->next release {res[7]:.2f}", flush=True)
