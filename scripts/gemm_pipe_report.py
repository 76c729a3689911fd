"""SURVEY 8(d) headline: duration-weighted int8 tensor-pipe utilisation of the decoder GEMMs.

usage: python scripts/gemm_pipe_report.py launches.csv [--preset small-aan] [--budget 8192]
                                          [--mcr 4096] [--out report.md]

Input: an ncu launch list of ONE translation job (scripts/job_once.py under
`ncu --nvtx --nvtx-include job/ --metrics gpu__time_duration.sum,
sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active --csv`).

- Launches before the first k_decode_init of a wave are the encoder's; the rest are decoder steps.
- Decoder GEMM classes by kernel template (k_gemm_i8 / k_gemm_pers / k_gemm_sab) + launch order: EPI 5 = output projection + argmax;
  RELU_Q (EPI 2) with N = F (grid.x * BN, or the persistent kernel) = FFN1; the first F32 GEMM
  after an FFN1 = FFN2; every other decoder GEMM = a d x d projection (AAN FFN, gates, source q/o).
- useful-ops % = sum 2*M*N*K over the job (M = live rows of each step, from the schedule) /
  (sum of the class's ncu durations x int8 peak).  ncu times are serialised and cold-cache, so the
  absolute durations are upper bounds; the shares are what the launch list is good for.
"""
import argparse
import collections
import csv
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def load(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[h]
    col = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Grid Size", "Metric Name", "Metric Unit", "Metric Value")}
    by_id = collections.OrderedDict()
    for r in rows[h + 1:]:
        if len(r) < len(hdr):
            continue
        k = by_id.setdefault(int(r[col["ID"]]), {"name": r[col["Kernel Name"]], "grid": r[col["Grid Size"]]})
        v = float(r[col["Metric Value"]].replace(",", "")) if r[col["Metric Value"]] not in ("", "n/a") else 0.0
        if r[col["Metric Name"]] == "gpu__time_duration.sum":
            k["us"] = v * SCALE.get(r[col["Metric Unit"]], 1.0)
        elif "pipe_tensor" in r[col["Metric Name"]] and "pct" in r[col["Metric Name"]]:
            k["pipe"] = v
    return list(by_id.values())


def classify(launches, F):
    phase = "enc"
    after_ffn1 = False
    for k in launches:
        n = k["name"]
        if "k_decode_init" in n:
            phase = "dec"
        if "k_embed_src" in n:
            phase = "enc"
        m = re.search(r"k_gemm_(i8|pers|sab)<(\d+), (\d+)>", n)
        if not m:
            k["cls"] = None
            continue
        pers, bn, epi = m.group(1) == "pers", int(m.group(2)), int(m.group(3))
        if m.group(1) == "sab":   # swap-AB: 128 output columns per CTA (the template's first
            bn = 128              # parameter is the row tile)
        gx = int(re.match(r"\((\d+)", k["grid"]).group(1)) if k["grid"].startswith("(") else 0
        N = None if pers else gx * bn
        if phase == "enc":
            k["cls"] = "encoder"
        elif epi == 5:
            k["cls"] = "output"
        elif epi == 2 and (pers or N == F):
            k["cls"] = "ffn1"
            after_ffn1 = True
            continue
        elif epi == 0 and after_ffn1:
            k["cls"] = "ffn2"
        else:
            k["cls"] = "dxd"
        after_ffn1 = False


def useful_ops(preset, budget, mcr):
    import numpy as np
    import synth
    from bench import live_rows_profile
    dims = synth.PRESETS[preset]
    sset = synth.newstest_set(seed=2014)
    rows = live_rows_profile(sset, budget, mcr)
    R = float(np.sum(rows))
    d, F, V, L = dims.d_model, dims.d_ffn, dims.vocab, dims.dec_layers
    # d x d GEMMs per layer: AAN FFN + gates + source q/o; self-attention: q|k|v (3) + o + q/o
    ndd = (dims.aan_ffn_depth + 2 * dims.aan_gate + 2) if dims.decoder == 1 else 6
    enc_tok = float(sset.lengths.sum())
    return {"dxd": 2.0 * R * d * d * ndd * L, "ffn1": 2.0 * R * d * F * L, "ffn2": 2.0 * R * F * d * L,
            "output": 2.0 * R * d * V,
            "encoder": 2.0 * enc_tok * (4 * d * d + 2 * d * F) * dims.enc_layers + 2.0 * enc_tok * d * 2 * d * L}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--preset", default="small-aan")
    ap.add_argument("--budget", type=int, default=8192)
    ap.add_argument("--mcr", type=int, default=4096)
    ap.add_argument("--out", default=None)
    ap.add_argument("--json", default=None, help="also write the figures as JSON (bench.py reads it)")
    ap.add_argument("--workload", default=None, help="bench workload name recorded in the JSON")
    a = ap.parse_args()
    import synth
    dims = synth.PRESETS[a.preset]
    L = load(a.csv)
    classify(L, dims.d_ffn)
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
    bf16 = float(peaks["bf16_tflops"])
    peak_ops = 2.0 * bf16 * 1e12
    ops = useful_ops(a.preset, a.budget, a.mcr)
    tot_us = sum(k.get("us", 0.0) for k in L)
    dec_us = 0.0
    seen_dec = False
    for k in L:
        seen_dec = seen_dec or "k_decode_init" in k["name"]
        if seen_dec:
            dec_us += k.get("us", 0.0)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for k in L:
        if k.get("cls"):
            g = agg[k["cls"]]
            g[0] += 1
            g[1] += k.get("us", 0.0)
            g[2] += k.get("us", 0.0) * k.get("pipe", 0.0)
    dec_cls = ["dxd", "ffn1", "ffn2", "output"]
    dec_t = sum(agg[c][1] for c in dec_cls)
    dec_pipe = sum(agg[c][2] for c in dec_cls) / dec_t if dec_t else 0.0
    lines = [f"# Decoder-GEMM tensor-pipe report ({a.preset}, budget {a.budget}, max_concurrent_rows {a.mcr})",
             f"source: {a.csv} ({len(L)} launches, {tot_us / 1e3:.1f} ms serialised ncu time; "
             f"int8 peak {peak_ops / 1e12:.0f} TOP/s = 2 x measured bf16)", "",
             f"**Headline (SURVEY 8(d)): decoder-GEMM tensor-pipe utilisation, duration-weighted = {dec_pipe:.2f}%**", "",
             "| class | launches | ncu time (ms) | share of decode time | tensor-pipe % (dur.-weighted) | useful ops (TOP) | useful-ops % of peak |",
             "|---|---|---|---|---|---|---|"]
    for c in dec_cls + ["encoder"]:
        n, t, tp = agg[c]
        if n == 0:
            continue
        share = t / dec_us if c != "encoder" and dec_us else float("nan")
        u = ops.get(c, 0.0)
        lines.append(f"| {c} | {n} | {t / 1e3:.2f} | {share * 100:.1f}% | {tp / t if t else 0:.2f} | "
                     f"{u / 1e12:.3f} | {100 * u / (t * 1e-6 * peak_ops) if t else 0:.2f}% |")
    lines += ["", f"Decoder GEMM kernels take {100 * dec_t / dec_us:.1f}% of the decode's serialised kernel time "
              f"({dec_t / 1e3:.1f} of {dec_us / 1e3:.1f} ms)."]
    txt = "\n".join(lines)
    print(txt)
    if a.out:
        open(a.out, "w").write(txt + "\n")
    if a.json:
        per = {}
        for c in dec_cls + ["encoder"]:
            n, t, tp = agg[c]
            if n:
                per[c] = {"launches": n, "ncu_ms": t / 1e3, "tensor_pipe_pct": tp / t if t else 0.0,
                          "useful_ops_pct": 100 * ops.get(c, 0.0) / (t * 1e-6 * peak_ops) if t else 0.0}
        dec_ops = sum(ops.get(c, 0.0) for c in dec_cls)
        json.dump({"workload": a.workload, "preset": a.preset, "budget": a.budget, "mcr": a.mcr,
                   "source": a.csv, "launches": len(L),
                   "decoder_gemm_tensor_pipe_pct": dec_pipe,
                   "decoder_gemm_useful_ops_pct": 100 * dec_ops / (dec_t * 1e-6 * peak_ops) if dec_t else 0.0,
                   "decoder_gemm_share_of_decode_time": dec_t / dec_us if dec_us else 0.0,
                   "per_class": per, "int8_peak_tops": peak_ops / 1e12},
                  open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
