#!/usr/bin/env python
"""Benchmark: batched greedy int8 decoding of a distilled AAN student (arXiv 1805.12096).

One "step" = one pass of the whole hot path over one batch of synthetic input: the
newstest2014-shaped set (3003 sentences, 62,954 source tokens), sorted by
length and cut into >= 8192-word batches, encoded and greedily decoded
(max_len = source length) with every product in int8 on the tensor cores.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mnmt|reference]
                    [--workload W] [--scaling weak|strong]

The default workload is BASELINE.json configs[3]: the big student (d 1024, F 4096, H 16,
plain self-attention decoder), greedy, on the newstest-shaped set.  N > 1: one process per
GPU over NCCL; without torchrun's environment `--gpus N` re-launches itself under
`torch.distributed.run`.  weak (default): every rank decodes its own newstest-shaped set;
strong: one set is length-sorted and dealt round-robin over the ranks.  The
ids of every rank are all-gathered and put in input order on rank 0 inside the timed region
(A11).  Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import re
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "target words/sec greedy decode at 1/2/4/8 B200; int8 tensor-pipe % of peak"
UNIT = "target words/s"
WORKLOADS = {
    # name: (preset, word budget, BASELINE.json config)
    "small-aan-newstest-8192w": ("small-aan", 8192, "configs[1]"),
    "tiny192-aan-newstest-8192w": ("tiny192-aan", 8192, "configs[0] model"),
    "base-newstest-8192w": ("base", 8192, "configs[2] self-attention"),
    "base-aan-newstest-8192w": ("base-aan", 8192, "configs[2] AAN"),
    "big-newstest-8192w": ("big", 8192, "configs[3]"),
}
DEFAULT_WORKLOAD = "big-newstest-8192w"   # BASELINE.json configs[3]: the metric's own config
# Per-workload launch options (scheduling only: ids are identical for every setting), from the
# green_sms x lane_tiers sweep on one B200 (profiles/r1_sweep_green_tiers.txt): the critical
# lane's SM partition pays off for the smaller students and costs the big one (its bulk lanes
# need every SM).
# smallm / smallm_kmax: the small-M (IDP4A, <= 32 live rows) GEMM path's row bound and deepest K
# per workload, from the A/B in profiles/r1_ab_smallm_*.txt (small-aan: +2 % with FFN2's K = 2048
# included; the others neutral or slower, so off; big with K <= 1024 and the <= 1 MB d x d maps:
# 91.5 -> 90.8 ms per job in round 2 (profiles/r2_sweep_big_options.txt)).
# sab: row bound of the swap-AB tcgen05 GEMM (weights as the 128-row MMA operand, live rows as
# N = 16 / 32 / 64; profiles/r2_sab_enc_ab.txt): big 88.9-89.5 -> 86.3-87.4 ms per job with sab 64
# and the IDP4A path off.  Every workload now runs its small-row decoder GEMMs on the tensor cores
# (sab, smallm 0): on the final build the IDP4A path is within 0.2-0.4 % of it for the AAN students
# (profiles/r2_tensor_core_small_rows.txt), and these products are dense contractions.
# attn_tma_self: self-attention decoders through the TMA-tiled kernels (profiles/r2_attn_tma_ab.txt,
# after the V tiles started reusing the K buffers: big 99.1-99.4 / 100.1-100.2 / 97.7-97.8 ms per
# job for 0 / 1 / 2, base self-attention 59.9 / 59.2 / 56.4 ms): 2.
WORKLOAD_OPTS = {
    "small-aan-newstest-8192w": {"lanes": 3, "green_sms": 48, "lane_tiers": 40, "smallm": 0, "smallm_kmax": 2048,
                                 "attn_tma_self": 2, "sab": 32},
    "tiny192-aan-newstest-8192w": {"lanes": 3, "green_sms": 56, "lane_tiers": 40, "smallm": 0, "smallm_kmax": 512,
                                   "attn_tma_self": 2, "sab": 32},
    "base-newstest-8192w": {"lanes": 3, "green_sms": 24, "lane_tiers": 40, "smallm": 0, "smallm_kmax": 512,
                            "attn_tma_self": 2, "sab": 32},
    "base-aan-newstest-8192w": {"lanes": 3, "green_sms": 40, "lane_tiers": 35, "smallm": 0, "smallm_kmax": 512,
                                "attn_tma_self": 2, "sab": 32},
    "big-newstest-8192w": {"lanes": 2, "green_sms": 0, "lane_tiers": 15, "smallm": 0, "smallm_kmax": 1024,
                           "attn_tma_self": 2, "sab": 64},
}
L2_FLUSH_BYTES = 512 << 20   # > 126 MB L2


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return {"hbm_gbs": float(d["hbm_gbs"]), "bf16_tflops": float(d["bf16_tflops"]),
                "bf16_tflops_sustained": float(d.get("bf16_tflops_sustained", d["bf16_tflops"])),
                "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "source": "fallback (B200_PROFILING.md)"}


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        loaded = [s for s in sm if smax and s > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------- oracle legs
def _oracle_run(om, subset, beam, sl=None):
    """Target words of one oracle pass (beam > 1: words of each sentence's best hypothesis;
    sl: the shortlist of every sentence's word-budget batch, decoded batch by batch)."""
    if sl is not None:
        return _oracle_run_sl(om, subset, *sl)
    if beam > 1:
        return sum(len(h[0][0]) if h else 0 for h in om.beam_many(subset, beam, 0))
    return sum(len(o) for o in om.decode_many(subset, 0))


def _oracle_run_sl(om, subset, bb_of, lists):
    """F2 oracle leg: the sample's sentences grouped by their word-budget batch, each group
    decoded over that batch's shortlist (orc_decode_many_sl)."""
    idx = subset.idx
    words = 0
    for b in sorted(set(bb_of[idx].tolist())):
        sub = subset.sset.subset(idx[bb_of[idx] == b])
        words += sum(len(o) for o in om.decode_many_sl(sub, lists[b], 0))
    return words


class _Sample:
    """A subset that remembers its indices (for the shortlist leg)."""
    def __init__(self, sset, idx):
        self.sset, self.idx = sset, np.asarray(idx)
        sub = sset.subset(self.idx)
        self.max_len, self.lengths = sub.max_len, sub.lengths


def oracle_shortlists(sset, dims, budget, freq, lex):
    """Per sentence its word-budget batch and per batch its shortlist."""
    import oracle.oracle as O
    order, off = O.batch_by_words(sset.lengths, budget)
    bb_of = np.empty(sset.n, np.int64)
    lists = []
    for b in range(len(off) - 1):
        rows = order[off[b]:off[b + 1]]
        bb_of[rows] = b
        lists.append(O.build_shortlist(dims.vocab, freq, lex, sset.subset(rows).ids,
                                       eos=dims.eos_id, unk=1))
    return bb_of, lists


def oracle_sample(sset, dims, weights, seconds: float, seed: int = 99, beam: int = 1, sl=None):
    """Decode a seeded random sample of the workload with the oracle, sized to ~`seconds`.
    Returns (target words/s, threads, description)."""
    import oracle.oracle as O
    om = O.OracleModel(dims, weights)
    if sl is not None:
        return _oracle_sample_sl(om, O, sset, seconds, seed, sl)
    threads = O.max_threads()
    rng = np.random.default_rng(seed)
    perm = rng.permutation(sset.n)
    probe = sset.subset(perm[:max(threads, 8)])
    t0 = time.perf_counter()
    w_probe = _oracle_run(om, probe, beam)
    dt = time.perf_counter() - t0
    rate = w_probe / max(dt, 1e-9)
    mean_len = float(np.mean(probe.max_len))
    n = int(min(sset.n, max(len(probe.max_len), rate * seconds / max(mean_len, 1.0))))
    samp = sset.subset(perm[:n])
    t0 = time.perf_counter()
    words = _oracle_run(om, samp, beam)
    dt = time.perf_counter() - t0
    mode = "greedy" if beam <= 1 else f"beam-{beam}"
    desc = (f"oracle {mode} decode of {n} of {sset.n} sentences (seeded random sample, "
            f"{int(samp.lengths.sum())} source / {words} target words, one batch per sentence, "
            f"OpenMP over sentences) in {dt:.1f} s")
    return words / dt, threads, desc, dt


def _oracle_sample_sl(om, O, sset, seconds, seed, sl):
    threads = O.max_threads()
    perm = np.random.default_rng(seed).permutation(sset.n)
    probe = _Sample(sset, perm[:max(threads, 8)])
    t0 = time.perf_counter()
    rate = _oracle_run(om, probe, 1, sl) / max(time.perf_counter() - t0, 1e-9)
    n = int(min(sset.n, max(len(probe.idx), rate * seconds / max(float(np.mean(probe.max_len)), 1.0))))
    samp = _Sample(sset, perm[:n])
    t0 = time.perf_counter()
    words = _oracle_run(om, samp, 1, sl)
    dt = time.perf_counter() - t0
    desc = (f"oracle greedy decode restricted to each sentence's batch shortlist (P:L85) of {n} of "
            f"{sset.n} sentences (seeded random sample, {int(samp.lengths.sum())} source / {words} "
            f"target words, OpenMP over sentences) in {dt:.1f} s")
    return words / dt, threads, desc, dt


def run_reference(args, dims, weights, sset, workload_cfg):
    """`--impl reference`: the CPU oracle as it stands, timed on the host cores."""
    import oracle.oracle as O
    O.build()
    om = O.OracleModel(dims, weights)
    threads = O.max_threads()
    rng = np.random.default_rng(123)
    perm = rng.permutation(sset.n)
    # size one step to ~8 s of CPU work
    probe = sset.subset(perm[:max(threads, 8)])
    t0 = time.perf_counter()
    rate = _oracle_run(om, probe, args.beam) / max(time.perf_counter() - t0, 1e-9)
    n = int(min(sset.n, max(len(probe.max_len), rate * 8.0 / max(float(np.mean(probe.max_len)), 1.0))))
    samp = sset.subset(perm[:n])
    for _ in range(args.warmup):
        _oracle_run(om, samp, args.beam)
    t0 = time.perf_counter()
    words = 0
    for _ in range(args.steps):
        words += _oracle_run(om, samp, args.beam)
    dt = time.perf_counter() - t0
    value = words / dt
    desc = (f"oracle {'greedy' if args.beam <= 1 else f'beam-{args.beam}'} decode of the same {n}-sentence seeded sample of the workload per step "
            f"({int(samp.lengths.sum())} source words)")
    line = {
        "impl": "reference", "metric": metric_name(args.beam, False, bool(args.kv_bf16)), "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int8/f32/f64",
        "data": "synthetic (seeded random-init weights, newstest2014-shaped ids)",
        "config": workload_cfg,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ---------------------------------------------------------------------------- roofline legs
def time_kernel(fn, iters: int, stream):
    """Average device time of one launch: `iters` launches captured in a CUDA graph (so host
    overhead of the op-level call is excluded), replayed, timed with CUDA events."""
    import torch
    for _ in range(3):
        fn(torch.cuda.current_stream())
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        cs = torch.cuda.current_stream()
        for _ in range(iters):
            fn(cs)
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    g.replay()
    e.record(stream)
    e.synchronize()
    return s.elapsed_time(e) / iters    # ms per launch


def live_rows_profile(sset, budget, max_concurrent_rows=0):
    """Live decode rows at every sequential step (max_len = S_i, no EOS), following the
    library's schedule: word-budget batches, co-scheduled in waves of <= max_concurrent_rows."""
    from paper_1805_12096_b200 import mnmt as M
    order, off = M.batch_by_words(sset.lengths, budget)
    nb = len(off) - 1
    rows = []
    b = 0
    while b < nb:
        e = b + 1
        if max_concurrent_rows > 0:
            while e < nb and off[e + 1] - off[b] <= max_concurrent_rows:
                e += 1
        ml = sset.max_len[order[off[b]:off[e]]]
        for t in range(1, int(ml.max()) + 1):
            rows.append(int(np.sum(ml >= t)))
        b = e
    return rows


def live_rows_profile_waves(sset, budget, max_concurrent_rows=0):
    """The decode waves of the library's schedule (lists of word-budget batch indices), for the
    config description: stable length sort, batches closed at >= budget words (R17)."""
    L = np.asarray(sset.lengths)[np.argsort(sset.lengths, kind="stable")]
    off, acc = [0], 0
    for i, x in enumerate(L):
        acc += int(x)
        if acc >= budget:
            off.append(i + 1)
            acc = 0
    if off[-1] != len(L):
        off.append(len(L))
    nb = len(off) - 1
    waves, b = [], 0
    while b < nb:
        e = b + 1
        if max_concurrent_rows > 0:
            while e < nb and off[e + 1] - off[b] <= max_concurrent_rows:
                e += 1
        waves.append(list(range(b, e)))
        b = e
    return waves


def roofline_out_gemm(dims, weights, sset, budget, peaks, stream, mcr, beam=0, fused=1,
                      n_cols=None):
    """A9: output projection fused with argmax (beam > 0: with the beam-search log-sum-exp +
    top-8 epilogue, EPI_TOPK, at beam x the mean live-row count), at the workload's mean
    live-row count (n_cols: the mean shortlist size, F2)."""
    import torch
    from paper_1805_12096_b200 import mnmt as M
    rows = live_rows_profile(sset, budget, mcr)
    Mr = int(round(np.mean(rows) * max(1, beam)))
    d, V = dims.d_model, dims.vocab
    dev = torch.device("cuda", torch.cuda.current_device())
    E = torch.from_numpy(weights["emb.E"]).to(dev)
    qE = torch.empty((V, d), dtype=torch.int8, device=dev)
    M.op_quantize(E.data_ptr(), V * d, dims.clip, qE.data_ptr(), stream)
    x = torch.randn((Mr, d), device=dev)
    qa = torch.empty((Mr, d), dtype=torch.int8, device=dev)
    M.op_quantize(x.data_ptr(), Mr * d, dims.clip, qa.data_ptr(), stream)
    b = torch.from_numpy(weights["out.b"]).to(dev)
    if beam and fused:
        part_ld = 2 * ((V + 255) // 256)
        keys = torch.empty(Mr * part_ld * M.TOPK_RECORD_BYTES, dtype=torch.uint8, device=dev)
        epi = M.EPI_TOPK
    elif beam:   # materialised logits (beam_fused = 0): the GEMM writes fp32 [rows x V]
        keys = torch.empty((Mr, V), dtype=torch.float32, device=dev)
        epi = M.EPI_F32
    else:
        keys = torch.zeros(Mr, dtype=torch.int64, device=dev)
        epi = M.EPI_ARGMAX

    N = int(n_cols) if n_cols else V

    def fn(st):
        M.op_gemm_i8(qa.data_ptr(), qE.data_ptr(), Mr, N, d, b.data_ptr(), dims.clip,
                     epi, keys.data_ptr(), None, beam if (beam in (2, 4) and fused) else 0, st)
    ms = time_kernel(fn, 200, stream)
    ops = 2.0 * Mr * N * d
    peak = 2.0 * peaks["bf16_tflops"]          # int8 dense = 2x bf16 (nominal 4.5 / 2.25)
    ach = ops / (ms * 1e-3) / 1e12
    name = (f"k_gemm_i8<256, EPI_TOPK{beam if beam in (2, 4) else ''}> (A9 beam output GEMM + "
            f"fp64 log-sum-exp + top-{beam if beam in (2, 4) else 8})" if beam and fused
            else "k_gemm_i8<EPI_F32> (A9 beam output GEMM writing fp32 logits)" if beam
            else "k_gemm_i8<EPI_ARGMAX> (A9 output GEMM + argmax" + (", shortlist)" if n_cols else ")"))
    return {"kernel": name, "bound": "tensor",
            "achieved": ach, "peak": peak, "unit": "TOP/s (int8)", "frac": ach / peak,
            "traffic": None, "shape": f"M={Mr} (mean live rows/step) N={N} K={d}",
            "ms_per_launch": ms, "launches_per_step": len(rows),
            "ms_per_step_est": ms * len(rows) * 1.0,
            "peak_source": f"{peaks['source']} bf16 burst x2"}


def roofline_dxd_gemm(dims, sset, budget, peaks, stream, mcr, mult=1):
    """A6-A7: the decoder's d x d projections (AAN FFN, gates, source q/o): 6 per layer per step,
    at the workload's mean live-row count."""
    import torch
    from paper_1805_12096_b200 import mnmt as M
    rows = live_rows_profile(sset, budget, mcr)
    Mr = max(1, int(round(np.mean(rows) * mult)))   # mult: beam (hypotheses per sentence)
    d = dims.d_model
    dev = torch.device("cuda", torch.cuda.current_device())
    A = torch.randint(-127, 128, (Mr, d), dtype=torch.int8, device=dev)
    W = torch.randint(-127, 128, (d, d), dtype=torch.int8, device=dev)
    b = torch.zeros(d, device=dev)
    out = torch.empty((Mr, d), device=dev)

    def fn(st):
        M.op_gemm_i8(A.data_ptr(), W.data_ptr(), Mr, d, d, b.data_ptr(), dims.clip, M.EPI_F32,
                     out.data_ptr(), None, 0, st)
    ms = time_kernel(fn, 200, stream)
    ops = 2.0 * Mr * d * d
    peak = 2.0 * peaks["bf16_tflops"]
    ach = ops / (ms * 1e-3) / 1e12
    per_step = 6 * dims.dec_layers if dims.decoder == 1 else 5 * dims.dec_layers
    # the library's tile choice (gemm_i8.cu launch_gemm_i8): 32-wide tiles when the 64-wide grid
    # fills less than half of the SMs and K <= 512, else 64 (N = d, small row counts)
    bn = 32 if (((d + 63) // 64) * ((Mr + 127) // 128) * 2 <= 148 and d <= 512) else 64
    return {"kernel": f"k_gemm_i8<{bn}, EPI_F32> (decoder d x d projections)", "bound": "tensor",
            "achieved": ach, "peak": peak, "unit": "TOP/s (int8)", "frac": ach / peak,
            "traffic": None, "shape": f"M={Mr} (mean live rows/step) N={d} K={d}",
            "ms_per_launch": ms, "launches_per_step": len(rows) * per_step,
            "ms_per_step_est": ms * len(rows) * per_step,
            "peak_source": f"{peaks['source']} bf16 burst x2"}


def roofline_src_attn(dims, sset, budget, peaks, stream, mcr, mult=1):
    """A7: source attention over the fp32 (kv_bf16: bf16, F3) K/V cache, rows = the workload's
    mean live rows per step, drawn (seeded) from the set so the source-length mix matches.
    Cold: consecutive launches rotate over copies of K/V whose total exceeds the 126 MB L2, so
    every launch streams its K/V from HBM (as in the job, where the K/V of six layers and
    thousands of rows cannot stay L2-resident)."""
    import torch
    from paper_1805_12096_b200 import mnmt as M
    rows = live_rows_profile(sset, budget, mcr)
    n_rows = max(1, int(round(np.mean(rows) * mult)))
    idx = np.random.default_rng(3).choice(sset.n, size=n_rows, replace=n_rows > sset.n)
    L = sset.lengths[idx].astype(np.int32)
    starts = np.concatenate([[0], np.cumsum(L)[:-1]]).astype(np.int32)
    d, H = dims.d_model, dims.n_heads
    n = len(idx)
    dev = torch.device("cuda", torch.cuda.current_device())
    kv16 = bool(getattr(dims, "kv_bf16", 0))
    one = int(L.sum()) * 2 * d * (2 if kv16 else 4)
    copies = max(2, int(np.ceil(384e6 / max(one, 1))))        # > 3x L2 in total
    kvs = []
    for _ in range(copies):
        kv = torch.randn((int(L.sum()), 2 * d), device=dev)
        kvs.append(kv.to(torch.bfloat16) if kv16 else kv)
    q = torch.randn((n, d), device=dev)
    st, ln = torch.from_numpy(starts).to(dev), torch.from_numpy(L).to(dev)
    oq = torch.empty((n, d), dtype=torch.int8, device=dev)
    it = [0]

    rows_kv, smax = int(L.sum()), int(L.max())

    def fn(s_):
        kv = kvs[it[0] % copies]
        it[0] += 1
        if kv16:
            M.op_attention_bf16(q.data_ptr(), d, kv.data_ptr(), 2 * d, 0, d, st.data_ptr(), ln.data_ptr(),
                                n, d, H, dims.clip, oq.data_ptr(), None, s_)
        else:   # the decode path's kernel choice (k_attn_tma for d_h = 32 / 64)
            M.op_src_attention(q.data_ptr(), d, kv.data_ptr(), rows_kv, 2 * d, 0, d, st.data_ptr(),
                               ln.data_ptr(), smax, n, d, H, dims.clip, oq.data_ptr(), None, s_)
    ms = time_kernel(fn, 200, stream)
    # K,V (fp32 or bf16) + q fp32 + codes
    bytes_ = float((4 if kv16 else 8) * d * L.sum() + n * (4 * d + d))
    ach = bytes_ / (ms * 1e-3) / 1e9
    peak = peaks["hbm_gbs"]
    tma = not kv16 and (d // H) in (32, 64)
    return {"kernel": ("k_attn_tma" if tma else "k_attn") + " (A7 source attention, fp64 accumulate" +
                      (", bf16 K/V)" if kv16 else ")"),
            "bound": "hbm",
            "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak, "traffic": None,
            "shape": f"rows={n} S_mean={L.mean():.1f} d={d} H={H} (one layer; K/V rotated over "
                     f"{copies} copies, {copies * one / 1e6:.0f} MB > L2)",
            "ms_per_launch": ms, "peak_source": peaks["source"]}


def roofline_ln(dims, sset, budget, peaks, stream, mcr, mult=1):
    """A6-A8: residual + LayerNorm + Q (k_ln, 3 per layer per step) at the mean live-row count;
    algorithmic bytes per row = x, delta (fp32) in, out (fp32) + codes out = 13 d."""
    import torch
    from paper_1805_12096_b200 import mnmt as M
    rows = live_rows_profile(sset, budget, mcr)
    n = max(1, int(round(np.mean(rows) * mult)))
    d = dims.d_model
    dev = torch.device("cuda", torch.cuda.current_device())
    copies = max(2, int(np.ceil(384e6 / (n * d * 8))))
    xs = [torch.randn((n, d), device=dev) for _ in range(copies)]
    ds = [torch.randn((n, d), device=dev) for _ in range(copies)]
    g = torch.ones(d, device=dev)
    b = torch.zeros(d, device=dev)
    out = torch.empty((n, d), device=dev)
    oq = torch.empty((n, d), dtype=torch.int8, device=dev)
    it = [0]

    def fn(s_):
        k = it[0] % copies
        it[0] += 1
        M.op_layernorm(xs[k].data_ptr(), ds[k].data_ptr(), None, None, g.data_ptr(), b.data_ptr(),
                       n, d, dims.ln_eps, dims.clip, out.data_ptr(), oq.data_ptr(), s_)
    ms = time_kernel(fn, 200, stream)
    bytes_ = 13.0 * d * n
    ach = bytes_ / (ms * 1e-3) / 1e9
    return {"kernel": "k_ln (A6-A8 residual + LayerNorm + Q)", "bound": "hbm", "achieved": ach,
            "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": ach / peaks["hbm_gbs"], "traffic": None,
            "shape": f"rows={n} d={d} (inputs rotated over {copies} copies > L2)",
            "ms_per_launch": ms, "launches_per_step": len(rows) * 3 * dims.dec_layers,
            "ms_per_step_est": ms * len(rows) * 3 * dims.dec_layers, "peak_source": peaks["source"]}


def ncu_traffic(key, shape, workload):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of this kernel from the committed
    `ncu --set full` capture of this workload (profiles/r2_ncu_full_kernels.json, written by
    scripts/ncu_full_summary.py from scripts/kernel_once.py runs), used only when the captured
    shape has the same row count as the one timed here."""
    path = os.path.join(ROOT, "profiles", "r2_ncu_full_kernels.json")
    try:
        with open(path) as f:
            rec = json.load(f)[f"{key}@{workload}"]
    except (OSError, KeyError, ValueError):
        return None, "no ncu capture of this kernel / workload"
    rows = lambda t: (re.search(r"(?:M|rows)=(\d+)", t) or [None, None])[1]
    if rows(rec["shape"]) != rows(shape):
        return None, f"ncu capture shape {rec['shape']} differs"
    return rec["traffic_bytes"], f"ncu --set full (cold L2), {rec['shape']}"


def gemm_pipe_record(workload):
    """SURVEY 8(d) headline: the duration-weighted decoder-GEMM tensor-pipe % of one job of this
    workload on this build, from the committed ncu pass (scripts/gemm_pipe_report.py --json)."""
    path = os.path.join(ROOT, "profiles", f"r2_decoder_gemm_pipe_{workload}.json")
    try:
        rec = json.load(open(path))
    except (OSError, ValueError):
        return None
    return {"decoder_gemm_tensor_pipe_pct": rec["decoder_gemm_tensor_pipe_pct"],
            "decoder_gemm_useful_ops_pct": rec["decoder_gemm_useful_ops_pct"],
            "decoder_gemm_share_of_decode_time": rec["decoder_gemm_share_of_decode_time"],
            "per_class": {k: {"tensor_pipe_pct": v["tensor_pipe_pct"], "useful_ops_pct": v["useful_ops_pct"]}
                          for k, v in rec["per_class"].items()},
            "source": os.path.relpath(path, ROOT) + " (ncu launch list of one job, serialised, cold L2)"}


# ---------------------------------------------------------------------------- main
def metric_name(beam: int, shortlist: bool = False, kv16: bool = False) -> str:
    if kv16 and beam <= 1 and not shortlist:
        return "target words/sec greedy decode with bf16 source keys/values (F3)"
    if shortlist:
        return "target words/sec greedy decode with batch vocabulary shortlist (100 frequent + 100 per source word)"
    return METRIC if beam <= 1 else f"target words/sec beam-{beam} decode (best hypothesis)"


def relaunch_under_torchrun(args):
    """`--gpus N` (N > 1) without torchrun's environment: re-run this command as N ranks."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mnmt", choices=["mnmt", "reference"])
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS))
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N > 1: weak = one newstest-shaped set per GPU (default); strong = one "
                         "set sharded round-robin in length order (SURVEY 8(e))")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-roofline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--beam", type=int, default=1,
                    help="1 (default): greedy decode, the headline; 2..8: beam search "
                         "(SURVEY 8(f) F1, mnmt_beam_translate); words = best hypothesis")
    ap.add_argument("--shortlist", action="store_true",
                    help="greedy decode with each batch's vocabulary shortlist (SURVEY 8(f) F2, "
                         "P:L85; synthetic Zipf tables, 100 frequent + 100 per source word)")
    ap.add_argument("--kv-bf16", action="store_true",
                    help="source keys / values rounded to bf16 (SURVEY 8(f) F3, src_kv_bf16 = 1)")
    ap.add_argument("--beam-fused", type=int, default=0,
                    help="beam search: 1 = log-sum-exp / top-k fused into the output GEMM epilogue")
    ap.add_argument("--lanes", type=int, default=None,
                    help="independent decoder lanes (streams) per GPU (scheduling only; default per workload)")
    ap.add_argument("--lane-tiers", type=int, default=None,
                    help="0: deal sentences round-robin to lanes; 10*p: contiguous length tiers "
                         "of equal sum S^p (scheduling only; default: per workload)")
    ap.add_argument("--green-sms", type=int, default=None,
                    help="SM partition (green context) of the critical lane; 0 = shared SMs "
                         "(default: per workload)")
    ap.add_argument("--pers-reserve", type=int, default=16,
                    help="SMs the persistent GEMMs of non-critical lanes leave free")
    ap.add_argument("--steps-per-graph", type=int, default=1,
                    help="decoder steps captured per CUDA graph (scheduling only)")
    ap.add_argument("--smallm", type=int, default=None,
                    help="row bound of the small-M IDP4A GEMM path (0 = tcgen05 always; "
                         "default per workload)")
    ap.add_argument("--smallm-kmax", type=int, default=None,
                    help="deepest K of the small-M path (default per workload)")
    ap.add_argument("--sab", type=int, default=None,
                    help="row bound of the swap-AB tcgen05 GEMM path (0 = off; default per workload)")
    ap.add_argument("--attn-tma-self", type=int, default=None,
                    help="self-attention through TMA tiles: 0 off, 1 split kernel, 2 all (default per workload)")
    ap.add_argument("--max-concurrent-rows", type=int, default=4096,
                    help="co-schedule consecutive >=budget-word batches in one decode wave "
                         "(scheduling only; 0 = one batch at a time)")
    ap.add_argument("--opt", action="append", default=[],
                    help="extra model option name=value (A/B runs; scheduling only)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    for k, v in WORKLOAD_OPTS.get(args.workload, {}).items():
        if getattr(args, k) is None:
            setattr(args, k, v)
    args.green_sms = 56 if args.green_sms is None else args.green_sms
    args.lanes = 3 if args.lanes is None else args.lanes
    args.lane_tiers = 40 if args.lane_tiers is None else args.lane_tiers

    if args.impl == "mnmt" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    preset, budget, cfg_ref = WORKLOADS[args.workload]
    dims = synth.PRESETS[preset]
    if args.kv_bf16:
        import dataclasses
        dims = dataclasses.replace(dims, name=dims.name + "-kvbf16", kv_bf16=1)
    scaling = args.scaling if world > 1 else "weak"
    mcr = args.max_concurrent_rows
    full = synth.newstest_set(seed=2014)
    waves = len(live_rows_profile_waves(full, budget, mcr))
    workload_cfg = {"workload": args.workload, "baseline_config": cfg_ref,
                    "student": f"{preset}: d={dims.d_model} F={dims.d_ffn} H={dims.n_heads} "
                               f"L={dims.enc_layers}+{dims.dec_layers} V={dims.vocab} "
                               f"decoder={'AAN' if dims.decoder else 'self-attn'}",
                    "sentences": synth.NEWSTEST_SENTENCES * (world if scaling == "weak" else 1),
                    "source_words": synth.NEWSTEST_TOKENS * (world if scaling == "weak" else 1),
                    "sharding": ("one newstest-shaped set per GPU (seed 2014 + rank)" if scaling == "weak"
                                 else "one newstest-shaped set, length-sorted, dealt round-robin over the GPUs"),
                    "word_budget": budget,
                    "schedule": (f"word-budget batches (>= {budget} words, P:L42) co-scheduled in waves of "
                                 f"<= {mcr} sentences: the 3003-sentence set decodes as {waves} wave(s), "
                                 f"split into {args.lanes} length-tiered lanes"),
                    "beam": args.beam, "beam_fused": args.beam_fused,
                    "src_kv": "bf16 (F3)" if args.kv_bf16 else "fp32",
                    "shortlist": "100 frequent + 100 per source word (synthetic Zipf tables, seed 85)" if args.shortlist else None,
                    "max_len": "source length", "parallelism": f"dp{world}",
                    "l2": "flushed between timed steps (512 MiB write)",
                    "max_concurrent_rows": mcr, "lanes": args.lanes,
                    "steps_per_graph": args.steps_per_graph, "smallm": args.smallm,
                    "smallm_kmax": args.smallm_kmax,
                    "lane_tiers": args.lane_tiers, "pers_reserve": args.pers_reserve,
                    "green_sms": args.green_sms, "attn_tma_self": args.attn_tma_self, "sab": args.sab,
                    "extra_options": args.opt,
                    "step_engine": "kernel-per-op CUDA graph per decoder step (PDL chained)"}

    if args.impl == "reference":
        if rank != 0:
            return
        weights = synth.make_weights(dims, seed=1)
        run_reference(args, dims, weights, full, workload_cfg)
        return

    import torch
    torch.cuda.set_device(local)
    dist_on = world > 1
    if dist_on:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        if world != args.gpus:
            raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE = {world}")
    from paper_1805_12096_b200 import dist as D
    from paper_1805_12096_b200 import mnmt as M

    weights = synth.make_weights(dims, seed=1)
    model = M.Model(dims, weights, device=local)
    for name, v in (("max_concurrent_rows", mcr), ("lanes", args.lanes),
                    ("steps_per_graph", args.steps_per_graph),
                    ("smallm", 32 if args.smallm is None else args.smallm),
                    ("smallm_kmax", 512 if args.smallm_kmax is None else args.smallm_kmax),
                    ("lane_tiers", args.lane_tiers), ("pers_reserve", args.pers_reserve),
                    ("green_sms", args.green_sms), ("beam_fused", args.beam_fused),
                    ("attn_tma_self", args.attn_tma_self or 0), ("sab", args.sab or 0)):
        model.set_option(name, v)
    for kv in args.opt:
        k, v = kv.split("=")
        model.set_option(k, int(v))
    # the rows this rank decodes, and the static gather / unshard plan of the whole job
    if scaling == "weak":
        sset = synth.newstest_set(seed=2014 + rank)
        n_each = sset.n
        shards = [np.arange(r * n_each, (r + 1) * n_each) for r in range(world)]
        ml_all = np.concatenate([synth.newstest_set(seed=2014 + r).max_len for r in range(world)]) \
            if world > 1 else sset.max_len
    else:
        shards = [D.shard_round_robin(full.lengths, r, world) for r in range(world)]
        sset = full.subset(shards[rank])
        ml_all = full.max_len
    use_sl = bool(args.shortlist)
    if use_sl:
        if args.beam > 1:
            raise SystemExit("--shortlist is greedy only")
        sl_freq, sl_lex = synth.shortlist_tables(dims.vocab, 100, 100, seed=85)
        model.set_shortlist(sl_freq, sl_lex)
    stream = torch.cuda.current_stream()
    dev = torch.device("cuda", local)
    ids_dev = torch.from_numpy(sset.ids).to(dev)
    beam = args.beam
    nb = max(1, beam)
    cap = int(sset.max_len.sum()) * nb
    out_dev = torch.zeros(max(cap, 1), dtype=torch.int32, device=dev)
    len_dev = torch.zeros(max(sset.n * nb, 1), dtype=torch.int32, device=dev)
    score_dev = torch.zeros(max(sset.n * nb, 1), dtype=torch.float32, device=dev)
    nhyp_dev = torch.zeros(max(sset.n, 1), dtype=torch.int32, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    plan = D.gather_plan(ml_all, shards) if dist_on and beam <= 1 else None
    unshard = D.DeviceUnshard(plan, dev) if plan is not None and rank == 0 else None
    launches_gather = 0

    def gather(flat_dev, lens_dev):
        """A11 across ranks: all_gather ids + lengths, input order on rank 0 (mnmt_op_gather_rows)."""
        gi, gl = D.all_gather_padded(flat_dev[:int(sset.max_len.sum())], lens_dev[:sset.n], plan)
        if unshard is not None:
            return unshard(gi, gl, stream)
        return None

    def step():
        if beam > 1:
            model.beam_translate_device(ids_dev.data_ptr(), sset.offsets, sset.max_len, budget,
                                        beam, out_dev.data_ptr(), cap, len_dev.data_ptr(),
                                        score_dev.data_ptr(), nhyp_dev.data_ptr(), stream)
        else:
            model.translate_device(ids_dev.data_ptr(), sset.offsets, sset.max_len, budget,
                                   out_dev.data_ptr(), cap, len_dev.data_ptr(), stream,
                                   shortlist=use_sl)
            if plan is not None:
                gather(out_dev, len_dev)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches_per_step = model.stats()["gpu_launches"] + (1 if unshard is not None else 0)
    if beam > 1:   # words of each sentence's best hypothesis
        words_rank = int((len_dev[:sset.n * nb].view(sset.n, nb)[:, 0] * (nhyp_dev[:sset.n] > 0)).sum().item())
    else:
        words_rank = int(len_dev[:sset.n].sum().item())

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if dist_on:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    for k in range(args.steps):
        flush.zero_()                       # untimed: L2 flush between timed steps
        ev[k][0].record(stream)
        step()
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    if dist_on:
        dist.barrier()
    clk = clocks.stop()
    ms_total = sum(a.elapsed_time(b) for a, b in ev)
    t = torch.tensor([ms_total, float(words_rank)], dtype=torch.float64, device=dev)
    if dist_on:
        tmax = t.clone()
        dist.all_reduce(tmax[0:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(tmax[1:2], op=dist.ReduceOp.SUM)
        t = tmax
    ms_max, words_total = float(t[0]), float(t[1])
    value = words_total * args.steps / (ms_max / 1000.0)
    if plan is not None and rank == 0:   # the gathered job equals the per-rank outputs
        assert int(unshard.lens.sum().item()) == int(words_total), "id gather lost rows"

    # ---- e2e: the public host-buffer call (H2D of ids, D2H of ids inside the timed region)
    def host_call():
        if beam > 1:
            return model.beam_translate(sset, budget, beam, stream)
        outs = model.translate(sset, budget, stream, shortlist=use_sl)
        if plan is not None:   # ids to the device, gathered, unsharded, back to rank 0's host
            flat, lens = D.pack_ids(outs, sset.max_len)
            res = gather(torch.from_numpy(flat).to(dev), torch.from_numpy(lens).to(dev))
            if res is not None:
                return D.split_rows(res[0].cpu().numpy(), res[1].cpu().numpy(), ml_all)
        return outs

    host_call()
    torch.cuda.synchronize()
    st = model.stats()
    e_ms = []
    for _ in range(args.e2e_steps):
        flush.zero_()
        torch.cuda.synchronize()
        if dist_on:
            dist.barrier()
        t0 = time.perf_counter()
        host_call()
        torch.cuda.synchronize()
        e_ms.append(1000 * (time.perf_counter() - t0))
    e = torch.tensor([sum(e_ms)], dtype=torch.float64, device=dev)
    if dist_on:
        dist.all_reduce(e, op=dist.ReduceOp.MAX)
    e2e_value = words_total * args.e2e_steps / (float(e[0]) / 1000.0)
    h2d, d2h = st["h2d_bytes"], st["d2h_bytes"]
    if plan is not None:
        h2d += int(sset.max_len.sum()) * 4 + sset.n * 4
        if rank == 0:
            d2h += plan.out_total * 4 + plan.n * 4

    roof = None
    cpu = None
    sl_lists = None
    if rank == 0 and not args.no_roofline:
        peaks = load_peaks()
        sl_lists = oracle_shortlists(sset, dims, budget, sl_freq, sl_lex) if use_sl else None
        n_cols = float(np.mean([len(x) for x in sl_lists[1]])) if use_sl else None
        cands = [roofline_out_gemm(dims, weights, sset, budget, peaks, stream, mcr,
                                   beam if beam > 1 else 0, args.beam_fused, n_cols),
                 roofline_src_attn(dims, sset, budget, peaks, stream, mcr, nb),
                 roofline_dxd_gemm(dims, sset, budget, peaks, stream, mcr, nb),
                 roofline_ln(dims, sset, budget, peaks, stream, mcr, nb)]
        cands[1]["launches_per_step"] = len(live_rows_profile(sset, budget, mcr)) * dims.dec_layers
        cands[1]["ms_per_step_est"] = cands[1]["ms_per_launch"] * cands[1]["launches_per_step"]
        keys = ("out", "attn16" if getattr(dims, "kv_bf16", 0) else "attn", "dxd", "ln")
        for key, c in zip(keys, cands):
            c["traffic"], c["traffic_source"] = ncu_traffic(key, c["shape"], args.workload)
        roof = max(cands, key=lambda c: c["ms_per_step_est"])
        roof["share_of_step_est"] = roof["ms_per_step_est"] / (ms_max / args.steps)
        roof["other"] = {c["kernel"]: {"frac": c["frac"], "ms_per_launch": c["ms_per_launch"],
                                       "ms_per_step_est": c["ms_per_step_est"]}
                         for c in cands if c is not roof}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sl = (sl_lists or oracle_shortlists(sset, dims, budget, sl_freq, sl_lex)) if use_sl else None
        v, cores, desc, _ = oracle_sample(sset, dims, weights, args.cpu_seconds, beam=beam, sl=sl)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc}

    if rank == 0:
        line = {
            "metric": metric_name(beam, use_sl, bool(args.kv_bf16)), "value": value, "unit": UNIT,
            "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None,
            "dtype": "int8 products (s32 acc), f32 activations, f64 reductions",
            "data": "synthetic (seeded random-init weights, newstest2014-shaped length-sorted ids)",
            "config": workload_cfg,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches_per_step * args.steps,
            "target_words_per_step": words_total,
            "decode_steps_per_gpu": st["decode_steps"], "batches_per_gpu": st["batches"],
            "clocks": clk, "roofline": roof, "cpu_baseline": cpu,
            "int8_tensor_pipe": gemm_pipe_record(args.workload) if beam <= 1 and not use_sl else None,
        }
        print(json.dumps(line))
    if dist_on:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
