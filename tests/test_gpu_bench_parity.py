"""P-2 / P-3 at the configurations bench.py times, against the CPU oracle.

* Teacher forcing through the whole mnmt_translate schedule (mnmt_translate_forced): the
  bench's workload model (seed-1 weights), its word budget and every launch option of
  bench.py's WORKLOAD_OPTS (3 length-tiered lanes, co-scheduled waves of <= 4096 sentences,
  SM partition, persistent-GEMM reserve, small-M GEMMs), every step replayed from its CUDA
  graph.  ~300 newstest-shaped sentences (every 10th in length order plus the longest, spans
  1..100): > 256 live rows in the first steps, a long tail that reaches the small-row paths.
  Every step's last-layer output and output codes, and x1/x2/x3 of every layer, come from a
  copy kernel captured in the step graphs.
* Free running on non-degenerate students (emb_scale 0.05, EOS bias raised): whole-sequence
  agreement, with a share of sentences ending at a mid-sentence EOS.

The summary of every run is appended to gpurun_out/parity/r2_parity.jsonl (copied to
profiles/ by the round script).
"""
import json
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import bench
import oracle.oracle as O
import synth
from tests.gpu_util import boundary_explained, check_forced_steps

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1805_12096_b200 import mnmt as M  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out", "parity", "r2_parity.jsonl")
THREADS = max(1, os.cpu_count() or 1)


def record(rec):
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    with open(OUT, "a") as f:
        f.write(json.dumps(rec) + "\n")


def bench_model(workload, weights):
    """The model with bench.py's launch options for `workload` (scheduling only)."""
    preset, budget, _ = bench.WORKLOADS[workload]
    dims = synth.PRESETS[preset]
    gm = M.Model(dims, weights)
    opts = {"max_concurrent_rows": 4096, "lanes": 3, "pers_reserve": 16, "steps_per_graph": 1}
    opts.update(bench.WORKLOAD_OPTS[workload])
    for k, v in opts.items():
        gm.set_option(k, v)
    return dims, gm, budget, opts


def stratified_newstest(step=10, longest=6):
    """Every `step`-th sentence of the newstest-shaped set in length order, plus the longest."""
    full = synth.newstest_set(seed=2014)
    order = np.argsort(full.lengths, kind="stable")
    idx = np.unique(np.concatenate([order[::step], order[-longest:]]))
    return full.subset(idx)


def forced_lengths(ss, seed, short=(3, 8), tail=24, tail_T=40):
    """Teacher-forcing lengths: most sentences a few steps, the `tail` longest sources up to
    tail_T steps (so late steps run with few live rows)."""
    rng = np.random.default_rng(seed)
    T = np.minimum(ss.lengths, rng.integers(short[0], short[1] + 1, size=ss.n))
    longest = np.argsort(ss.lengths, kind="stable")[-tail:]
    T[longest] = np.minimum(ss.lengths[longest], tail_T)
    return np.maximum(T, 1)


def oracle_traces(om, ss, forced, foff, layers=True):
    """Per-sentence oracle traces (teacher-forced unless forced=False), threads over sentences."""
    def one(i):
        src = ss.ids[ss.offsets[i]:ss.offsets[i + 1]]
        T = int(foff[i + 1] - foff[i])
        f = forced[foff[i]:foff[i + 1]] if forced is not False else None
        return om.decode_one(src, T, forced=f, trace=True, layers=layers)[1]
    with ThreadPoolExecutor(THREADS) as ex:
        return list(ex.map(one, range(ss.n)))


def rel_err(got, ref):
    """max |g - o| / max(|o|, rms(o_row)) (SURVEY 8(c).4 P-1 error measure), per element."""
    ref = ref.astype(np.float64)
    rms = np.sqrt(np.mean(ref * ref, axis=-1, keepdims=True))
    return float(np.max(np.abs(got.astype(np.float64) - ref) / np.maximum(np.abs(ref), np.maximum(rms, 1e-30))))


@pytest.mark.parametrize("workload", ["small-aan-newstest-8192w", "base-aan-newstest-8192w",
                                      "base-newstest-8192w", "big-newstest-8192w"])
def test_teacher_forced_bench_schedule(workload):
    preset = bench.WORKLOADS[workload][0]
    dims = synth.PRESETS[preset]
    w = synth.make_weights(dims, seed=1)            # bench.py's weights
    dims, gm, budget, opts = bench_model(workload, w)
    ss = stratified_newstest()
    T = forced_lengths(ss, seed=31)
    foff = np.concatenate([[0], np.cumsum(T)]).astype(np.int64)
    forced = synth.forced_targets(T.tolist(), seed=32, vocab=dims.vocab)
    mask = M.DUMP_DEC_OUT | M.DUMP_OUT_CODES | M.DUMP_LAYERS | M.DUMP_MARGIN
    ids, dumps = gm.decode_forced(ss, forced, foff, mask, budget=budget)
    st = gm.stats()
    om = O.OracleModel(dims, w)
    traces = oracle_traces(om, ss, forced, foff)
    qE = O.quantize(w["emb.E"])
    s = O.dequant_scale(dims.clip)
    tot = ex = fl = 0
    err_dec = err_layers = 0.0
    flips = unexplained = margin_diff = 0
    min_margin = float("inf")
    for i, tr in enumerate(traces):
        sl = slice(int(foff[i]), int(foff[i + 1]))
        err_dec = max(err_dec, rel_err(dumps["dec_out"][sl], tr["dec_out"]))
        err_layers = max(err_layers, rel_err(dumps["layers"][sl], tr["layer_out"]))
        flips += int(np.sum(dumps["out_codes"][sl] != tr["out_codes"]))
        unexplained += int(np.sum(boundary_explained(tr["dec_out"], tr["out_codes"], dumps["out_codes"][sl])))
        n_, e_, f_ = check_forced_steps(ids[sl], dumps["out_codes"][sl], tr, qE, s)
        tot += n_; ex += e_; fl += f_
        same = np.all(dumps["out_codes"][sl] == tr["out_codes"], axis=1)
        margin_diff += int(np.sum(dumps["margin"][sl][same] != tr["margin"][same]))
        min_margin = min(min_margin, float(np.min(tr["margin"])))
    rec = {"kind": "teacher-forced (mnmt_translate_forced, bench schedule)", "workload": workload,
           "options": opts, "word_budget": budget, "sentences": int(ss.n),
           "source_span_max": int(ss.lengths.max()), "steps_total": int(tot),
           "max_live_rows_step1": int(ss.n), "decode_steps": st["decode_steps"], "batches": st["batches"],
           "ids_identical": int(ex), "near_ties_flagged": int(fl), "ids_identical_pct": 100.0 * ex / tot,
           "max_rel_err_dec_out": err_dec, "max_rel_err_layers": err_layers,
           "output_code_flips": flips, "unexplained_code_flips": unexplained,
           "top2_margin_mismatches": margin_diff, "min_oracle_top2_margin": min_margin}
    record(rec)
    assert unexplained == 0, rec
    assert err_dec <= 1e-4 and err_layers <= 1e-4, rec
    assert ex + fl == tot, rec
    assert margin_diff == 0, rec


def eos_student(dims, seed=5, emb_scale=0.05, t_cross=8):
    """A student whose greedy outputs end at a mid-sentence EOS: E ~ U(-0.05, 0.05) (first
    tokens depend on the source), the EOS row of E set to the direction in which the oracle's
    last-layer output drifts over the first 16 steps (late minus early mean over 8 long
    sentences), and the EOS bias set so that EOS overtakes the top logit near step t_cross
    for the median probe sentence.  Built from oracle traces only (test input, not a method
    step)."""
    w = synth.make_weights(dims, seed=seed, emb_scale=emb_scale)
    om = O.OracleModel(dims, w)
    full = synth.newstest_set(seed=2014)
    order = np.argsort(full.lengths, kind="stable")
    probe = full.subset(order[-40::5])
    trs = oracle_traces(om, probe, False, np.arange(probe.n + 1, dtype=np.int64) * 16, layers=False)
    u = np.mean([t["dec_out"][10:16].mean(0) - t["dec_out"][:3].mean(0) for t in trs], axis=0)
    u = (u / np.sqrt(np.mean(u * u)) * emb_scale * 0.9).astype(np.float32)
    w["emb.E"] = w["emb.E"].copy()
    w["emb.E"][dims.eos_id] = u
    qE = O.quantize(w["emb.E"])
    s = O.dequant_scale(dims.clip)
    gaps = []
    for t in trs:
        qa = t["out_codes"][t_cross - 1].astype(np.int64)
        lg = s * (qE.astype(np.int64) @ qa).astype(np.float64) + w["out.b"]
        gaps.append(float(np.max(lg) - lg[dims.eos_id] + w["out.b"][dims.eos_id]))
    w["out.b"] = w["out.b"].copy()
    w["out.b"][dims.eos_id] = np.float32(np.median(gaps))
    return w


@pytest.mark.parametrize("workload", ["small-aan-newstest-8192w", "base-aan-newstest-8192w",
                                      "big-newstest-8192w"])
def test_free_running_nondegenerate(workload):
    """P-3: free-running greedy decode of a student built to end sentences at a mid-sentence
    EOS (eos_student), bench launch options, newstest-shaped sentences; every sentence
    identical to the oracle's."""
    preset = bench.WORKLOADS[workload][0]
    dims = synth.PRESETS[preset]
    w = eos_student(dims)
    eos_bias = float(w["out.b"][dims.eos_id])
    dims, gm, budget, opts = bench_model(workload, w)
    ss = stratified_newstest(step=15, longest=4)
    got = gm.translate(ss, budget)
    ref = O.OracleModel(dims, w).decode_many(ss, 0)
    same = [np.array_equal(a, b) for a, b in zip(got, ref)]
    mid = sum(0 < len(r) < m for r, m in zip(ref, ss.max_len))
    first_tokens = len(set(int(r[0]) for r in ref if len(r)))
    first_div = []
    for a, b in zip(got, ref):
        if not np.array_equal(a, b):
            k = next((j for j in range(min(len(a), len(b))) if a[j] != b[j]), min(len(a), len(b)))
            first_div.append(k)
    rec = {"kind": "free-running (mnmt_translate, bench options)", "workload": workload,
           "weights": "eos_student: seed 5, emb_scale 0.05, EOS row = drift direction, EOS bias %.3f" % eos_bias,
           "sentences": int(ss.n),
           "identical_pct": 100.0 * sum(same) / ss.n, "mid_sentence_eos_pct": 100.0 * mid / ss.n,
           "distinct_first_tokens": first_tokens, "first_divergence_steps": first_div,
           "target_words": int(sum(len(r) for r in ref))}
    record(rec)
    assert mid >= 0.1 * ss.n, rec
    assert all(same), rec


@pytest.mark.parametrize("workload", ["big-newstest-8192w", "base-newstest-8192w"])
def test_attn_f32_option_ids(workload):
    """The fp32 decoder-attention option (attn_f32, off by default; departs from R20): under teacher
    forcing through the bench schedule every per-step id equals the oracle's or is a near-tie explained
    by the step's output-code flips (check_forced_steps); free running on the EOS student the
    whole-sentence agreement is reported.  Intermediates are NOT held to 1e-4 (a context code that
    flips at a rounding boundary moves the next GEMM's output by s * w), so the option stays off."""
    preset = bench.WORKLOADS[workload][0]
    dims = synth.PRESETS[preset]
    w = synth.make_weights(dims, seed=1)
    dims, gm, budget, opts = bench_model(workload, w)
    gm.set_option("attn_f32", 1)
    ss = stratified_newstest()
    T = forced_lengths(ss, seed=31)
    foff = np.concatenate([[0], np.cumsum(T)]).astype(np.int64)
    forced = synth.forced_targets(T.tolist(), seed=32, vocab=dims.vocab)
    ids, dumps = gm.decode_forced(ss, forced, foff, M.DUMP_DEC_OUT | M.DUMP_OUT_CODES, budget=budget)
    om = O.OracleModel(dims, w)
    traces = oracle_traces(om, ss, forced, foff, layers=False)
    qE = O.quantize(w["emb.E"])
    s = O.dequant_scale(dims.clip)
    tot = ex = fl = 0
    err_dec = 0.0
    flips = 0
    for i, tr in enumerate(traces):
        sl = slice(int(foff[i]), int(foff[i + 1]))
        err_dec = max(err_dec, rel_err(dumps["dec_out"][sl], tr["dec_out"]))
        flips += int(np.sum(dumps["out_codes"][sl] != tr["out_codes"]))
        n_, e_, f_ = check_forced_steps(ids[sl], dumps["out_codes"][sl], tr, qE, s)
        tot += n_; ex += e_; fl += f_
    we = eos_student(dims)
    gm2 = bench_model(workload, we)[1]
    gm2.set_option("attn_f32", 1)
    ss2 = stratified_newstest(step=15, longest=4)
    got = gm2.translate(ss2, budget)
    ref = O.OracleModel(dims, we).decode_many(ss2, 0)
    same = [np.array_equal(a, b) for a, b in zip(got, ref)]
    rec = {"kind": "attn_f32 option (fp32 decoder attention; departs from R20)", "workload": workload,
           "options": dict(opts, attn_f32=1), "teacher_forced_steps": int(tot), "ids_identical": int(ex),
           "near_ties_flagged": int(fl), "ids_identical_pct": 100.0 * ex / tot,
           "max_rel_err_dec_out": err_dec, "output_code_flips": flips,
           "free_running_sentences": int(ss2.n), "free_running_identical_pct": 100.0 * sum(same) / ss2.n}
    record(rec)
    assert ex + fl == tot, rec
