"""How far the paper's CPU integer arithmetic departs from exact s32 accumulation (SURVEY 8(f)
F4; oracle only).  Greedy-decodes a seeded sample of the newstest-shaped set with the oracle
under arith 0 (exact s32, the GPU path), 1 (int8 codes, saturating int16 pair accumulation,
P:L94) and 2 (int16 codes x 2^10, wrapping int32 accumulation) and reports sentence /
token agreement with arith 0.

usage: python scripts/arith_departure.py [preset] [n_sentences] [emb_scale] > out.json"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import oracle.oracle as O  # noqa: E402

preset = sys.argv[1] if len(sys.argv) > 1 else "tiny192-aan"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 48
emb_scale = float(sys.argv[3]) if len(sys.argv) > 3 else 0.5
dims = synth.PRESETS[preset]
w = synth.make_weights(dims, seed=1, emb_scale=emb_scale)
ss = synth.newstest_set()
idx = np.random.default_rng(5).choice(ss.n, size=n, replace=False)
sub = ss.subset(idx)
res = {"preset": preset, "sentences": n, "emb_scale": emb_scale, "threads": O.max_threads()}
ref = None
for arith, name in ((0, "s32_exact"), (1, "int8_sat16_pairs"), (2, "int16_x1024_wrap32")):
    om = O.OracleModel(dims, w, arith=arith)
    t0 = time.perf_counter()
    out = om.decode_many(sub, 0)
    dt = time.perf_counter() - t0
    words = sum(len(o) for o in out)
    r = {"seconds": round(dt, 2), "target_words": words}
    if ref is None:
        ref = out
    else:
        same = sum(np.array_equal(a, b) for a, b in zip(out, ref))
        agree = 0
        for a, b in zip(out, ref):
            k = 0
            while k < min(len(a), len(b)) and a[k] == b[k]:
                k += 1
            agree += k
        r.update({"identical_sentences_pct": 100.0 * same / n,
                  "tokens_before_first_divergence_pct": 100.0 * agree / max(1, sum(len(b) for b in ref))})
    res[name] = r
print(json.dumps(res))
