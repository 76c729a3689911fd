"""Per-phase device time of the persistent step kernel at a small live-row count (uniform B x T)."""
import ctypes as C, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_1805_12096_b200 import mnmt as M
L = M.lib()
L.mnmt_debug_phase_times.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]
dims = synth.PRESETS["small-aan"]
m = M.Model(dims, synth.make_weights(dims, 1))
B = int(os.environ.get("B", 8))
m.set_option("profile_phases", 1); m.set_option("megakernel", 1)
for k, v in (a.split("=") for a in sys.argv[1:]):
    m.set_option(k, int(v))
ss = synth.uniform_set(B, 64, seed=5)
m.translate(ss, 1 << 30); m.translate(ss, 1 << 30)
avg = np.zeros(256, np.int64); ty = np.zeros(256, np.int32); n = np.zeros(1, np.int32)
L.mnmt_debug_phase_times(m.h, avg.ctypes.data, ty.ctypes.data, 256, n.ctypes.data)
names = ["GEMM", "EMBED", "LN", "ATTN", "FINISH"]
print(f"B={B}: {n[0]} phases, sum {avg[:n[0]].sum()/1e3:.1f} us/step")
print(" ".join(f"{names[ty[i]][0]}{avg[i]/1e3:.1f}" for i in range(n[0])))
