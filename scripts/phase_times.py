"""Per-phase average time of the persistent step kernel (lane 0), first-step and whole-job."""
import ctypes as C, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_1805_12096_b200 import mnmt as M
L = M.lib()

L.mnmt_debug_phase_times.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]
dims = synth.PRESETS[sys.argv[1] if len(sys.argv) > 1 else "small-aan"]
m = M.Model(dims, synth.make_weights(dims, 1))
ss = synth.newstest_set()
m.set_option("max_concurrent_rows", 4096); m.set_option("profile_phases", 1); m.set_option("megakernel", 1)
if len(sys.argv) > 2: m.set_option("rowlocal", int(sys.argv[2]))
names = ["GEMM", "EMBED", "LN", "ATTN", "FINISH"]
for cap in (1, 200):
    s2 = synth.SentenceSet(ss.ids, ss.offsets, np.minimum(ss.max_len, cap).astype(np.int32))
    m.translate(s2, 8192); m.translate(s2, 8192)
    avg = np.zeros(256, np.int64); ty = np.zeros(256, np.int32); n = np.zeros(1, np.int32)
    L.mnmt_debug_phase_times(m.h, avg.ctypes.data, ty.ctypes.data, 256, n.ctypes.data)
    print(f"--- max_len cap {cap}: {n[0]} phases, sum {avg[:n[0]].sum()/1e3:.1f} us/step")
    print(" ".join(f"{names[ty[i]][0]}{avg[i]/1e3:.1f}" for i in range(n[0])))
L.mnmt_debug_barrier_ns.restype = C.c_longlong
print("barrier ns (mode 0,1,2):", [L.mnmt_debug_barrier_ns(k, 2000) for k in (0, 1, 2)])
