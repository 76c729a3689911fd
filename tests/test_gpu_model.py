"""P-2/P-3/P-4: whole-pipeline parity of libmnmt against the CPU oracle.

  * teacher-forced: per-step argmax ids bit-exact (near-ties flagged only when explained by
    final-layer code flips), encoder output / source K,V / every decoder layer's x1,x2,x3
    equal to the oracle's up to last-bit double-rounding events;
  * free-running: whole-sequence agreement (required 100% on these sizes);
  * invariance: ids identical across word budgets, batch composition and order.
"""
import numpy as np
import pytest

import oracle.oracle as O
import synth
from synth import ModelDims
from tests.gpu_util import check_forced_steps

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1805_12096_b200 import mnmt as M  # noqa: E402

TINY_VARIANTS = [
    ModelDims("t-aan", 32, 64, 4, vocab=64, enc_layers=2, dec_layers=2),
    ModelDims("t-ffn1", 32, 64, 4, vocab=64, enc_layers=2, dec_layers=2, aan_ffn_depth=1),
    ModelDims("t-noffn-gate", 32, 64, 4, vocab=64, enc_layers=2, dec_layers=2, aan_ffn_depth=0),
    ModelDims("t-noffn-nogate", 32, 64, 4, vocab=64, enc_layers=2, dec_layers=2,
              aan_ffn_depth=0, aan_gate=0),
    ModelDims("t-self", 32, 64, 4, vocab=64, enc_layers=2, dec_layers=2, decoder=0),
    ModelDims("t-nobias-ragged-vocab", 48, 96, 4, vocab=50, enc_layers=1, dec_layers=3, out_bias=0),
    # d in {192, 256}: the paper-width head sizes (d_h = 24, 32)
    ModelDims("t192-aan", 192, 384, 8, vocab=1000, enc_layers=2, dec_layers=2),
    ModelDims("t192-ffn1", 192, 384, 8, vocab=1000, enc_layers=2, dec_layers=2, aan_ffn_depth=1),
    ModelDims("t256-noffn-gate", 256, 512, 8, vocab=1000, enc_layers=2, dec_layers=2, aan_ffn_depth=0),
    ModelDims("t256-self", 256, 512, 8, vocab=1000, enc_layers=2, dec_layers=2, decoder=0),
]


def pair(dims, seed):
    w = synth.make_weights(dims, seed=seed)
    return w, O.OracleModel(dims, w), M.Model(dims, w)


def forced_case(dims, n, lo, hi, T_lo, T_hi, seed):
    ss = synth.random_set(n, lo, hi, seed=seed, vocab=dims.vocab)
    rng = np.random.default_rng(seed + 1)
    T = rng.integers(T_lo, T_hi + 1, size=n)
    foff = np.zeros(n + 1, np.int64)
    foff[1:] = np.cumsum(T)
    forced = synth.forced_targets(T.tolist(), seed=seed + 2, vocab=dims.vocab)
    return ss, forced, foff


def run_forced_parity(dims, w, om, gm, ss, forced, foff, layers=True):
    mask = M.DUMP_ENC_OUT | M.DUMP_SRC_KV | M.DUMP_DEC_OUT | M.DUMP_OUT_CODES | M.DUMP_MARGIN
    if layers:
        mask |= M.DUMP_LAYERS
    ids, dumps = gm.decode_forced(ss, forced, foff, mask)
    qE = O.quantize(w["emb.E"])
    s = O.dequant_scale(dims.clip)
    tot = ex = fl = 0
    for i in range(ss.n):
        src = ss.ids[ss.offsets[i]:ss.offsets[i + 1]]
        T = int(foff[i + 1] - foff[i])
        f = forced[foff[i]:foff[i + 1]]
        oids, tr = om.decode_one(src, T, forced=f, trace=True, layers=layers)
        sl = slice(int(foff[i]), int(foff[i + 1]))
        if len(src):
            enc, kv = om.encode(src)
            a, b = int(ss.offsets[i]), int(ss.offsets[i + 1])
            np.testing.assert_allclose(dumps["enc_out"][a:b], enc, rtol=1e-6, atol=1e-6)
            np.testing.assert_allclose(dumps["src_kv"][:, a:b].transpose(0, 2, 1, 3), kv, rtol=1e-6, atol=1e-6)
        if T == 0:
            continue
        np.testing.assert_allclose(dumps["dec_out"][sl], tr["dec_out"], rtol=1e-5, atol=1e-5)
        if layers:
            np.testing.assert_allclose(dumps["layers"][sl], tr["layer_out"], rtol=1e-5, atol=1e-5)
        n_, e_, f_ = check_forced_steps(ids[sl], dumps["out_codes"][sl], tr, qE, s)
        tot += n_; ex += e_; fl += f_
        # top2_margin: identical wherever the step's output codes are (same s32 logits)
        same = np.all(dumps["out_codes"][sl] == tr["out_codes"], axis=1)
        assert np.array_equal(dumps["margin"][sl][same], tr["margin"][same]), i
    return tot, ex, fl


@pytest.mark.parametrize("dims", TINY_VARIANTS, ids=lambda d: d.name)
def test_tiny_teacher_forced(dims):
    w, om, gm = pair(dims, 11)
    ss, forced, foff = forced_case(dims, 9, 0, 13, 0, 17, seed=3)
    tot, ex, fl = run_forced_parity(dims, w, om, gm, ss, forced, foff)
    assert ex == tot, f"{tot - ex} flagged near-ties"


@pytest.mark.parametrize("lo,hi", [(30, 90), (60, 140)], ids=["split2", "split4"])
def test_long_sources_split_attention(lo, hi):
    """Long source spans take the split source-attention kernel (2 or 4 warps per (row, head),
    R25): every intermediate within tolerance of the oracle, ids bit-exact."""
    dims = TINY_VARIANTS[0]
    w, om, gm = pair(dims, 21)
    ss, forced, foff = forced_case(dims, 7, lo, hi, 2, 6, seed=9)
    tot, ex, fl = run_forced_parity(dims, w, om, gm, ss, forced, foff)
    assert ex == tot, f"{tot - ex} flagged near-ties"


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("dims", [d for d in TINY_VARIANTS if d.decoder == 0 and d.d_model == 256],
                         ids=lambda d: d.name)
def test_self_attention_tma(dims, mode):
    """Self-attention through the TMA-tiled kernels (option attn_tma_self: 1 = the split kernel for
    long decodes at <= 128 rows, 2 = every step; the step's k, v appended before the tensor copies
    read them): teacher-forced intermediates within tolerance of the oracle, ids bit-exact; and
    free-running ids with decodes long enough (70 steps) for the 2- and 4-warp splits."""
    w, om, gm = pair(dims, 11)
    gm.set_option("attn_tma_self", mode)
    ss, forced, foff = forced_case(dims, 9, 0, 13, 0, 17, seed=3)
    tot, ex, fl = run_forced_parity(dims, w, om, gm, ss, forced, foff)
    assert ex == tot, f"{tot - ex} flagged near-ties"
    ls = synth.random_set(12, 30, 70, seed=19, vocab=dims.vocab)
    ls.max_len[:] = np.random.default_rng(4).integers(60, 130, size=12)
    ref = om.decode_many(ls, 4)
    assert all(np.array_equal(a, b) for a, b in zip(gm.translate(ls, 1 << 20), ref))


@pytest.mark.parametrize("dims", TINY_VARIANTS, ids=lambda d: d.name)
def test_tiny_free_running(dims):
    w, om, gm = pair(dims, 12)
    ss = synth.random_set(17, 1, 15, seed=5, vocab=dims.vocab)
    ref = om.decode_many(ss, 4)
    got = gm.decode(ss)
    assert all(np.array_equal(a, b) for a, b in zip(got, ref))
    for k in (1, 3):                       # several decoder steps per CUDA graph
        gm.set_option("steps_per_graph", k)
        assert all(np.array_equal(a, b) for a, b in zip(gm.decode(ss), ref)), k
    gm.set_option("steps_per_graph", 1)


@pytest.mark.parametrize("dims", TINY_VARIANTS, ids=lambda d: d.name)
def test_small_m_gemms_teacher_forced(dims):
    """Small-M path (live rows <= the "smallm" bound: IDP4A k_gemm_smallm for the decoder's
    fp32 / code GEMMs, K split into 1, 2 or 4 segments by these widths) on and off: every intermediate within
    tolerance of the oracle, ids bit-exact, and the two paths' ids identical."""
    w, om, gm = pair(dims, 15)
    ss, forced, foff = forced_case(dims, 9, 0, 13, 0, 17, seed=8)
    got = {}
    for bound in (32, 16, 0):    # row bound of the small-M path (9 rows: on, on, off)
        gm.set_option("smallm", bound)
        tot, ex, fl = run_forced_parity(dims, w, om, gm, ss, forced, foff)
        assert ex == tot, (bound, f"{tot - ex} flagged near-ties")
        got[bound], _ = gm.decode_forced(ss, forced, foff, 0)
    gm.set_option("smallm", 32)
    assert np.array_equal(got[0], got[32]) and np.array_equal(got[0], got[16])


@pytest.mark.parametrize("preset", ["small-aan", "base"])
def test_small_m_gemms_paper_students(preset):
    """The paper's student widths (K = 256 / 512 / 2048: 4 and 8 K segments, the deep-K loop
    with smallm_kmax raised):
    teacher-forced layer dumps against the oracle and free-running ids equal to the oracle with
    the small-M path, and equal to the tcgen05 path's."""
    dims = synth.PRESETS[preset]
    w, om, gm = pair(dims, 16)
    gm.set_option("smallm_kmax", 2048)
    ss, forced, foff = forced_case(dims, 5, 1, 9, 1, 6, seed=10)
    tot, ex, fl = run_forced_parity(dims, w, om, gm, ss, forced, foff)
    assert ex == tot, f"{tot - ex} flagged near-ties"
    fs = synth.random_set(7, 1, 8, seed=12, vocab=dims.vocab)
    ref = om.decode_many(fs, 4)
    got = gm.decode(fs)
    assert all(np.array_equal(a, b) for a, b in zip(got, ref))
    gm.set_option("smallm", 0)
    assert all(np.array_equal(a, b) for a, b in zip(gm.decode(fs), ref))
    gm.set_option("smallm", 32)
    gm.set_option("smallm_kmax", 512)
    assert all(np.array_equal(a, b) for a, b in zip(gm.decode(fs), ref))


@pytest.mark.parametrize("smallm", [32, 0])
def test_big_student_teacher_forced(smallm):
    """big (d 1024, F 4096, H 16; K = 1024 / 4096): teacher-forced layer dumps against the oracle
    with the small-M IDP4A path taking every <= 32-row GEMM (8 K segments of 128 / 512 bytes;
    smallm_kmax / smallm_wmax raised) and with tcgen05 only (split-K clusters on FFN2, K = 4096,
    option split_k); ids bit-exact, every intermediate within tolerance."""
    dims = synth.PRESETS["big"]
    w, om, gm = pair(dims, 17)
    gm.set_option("smallm", smallm)
    gm.set_option("smallm_kmax", 4096)
    gm.set_option("smallm_wmax", 1 << 24)
    gm.set_option("split_k", 1 if smallm == 0 else 0)
    ss, forced, foff = forced_case(dims, 6, 1, 12, 1, 8, seed=11)
    tot, ex, fl = run_forced_parity(dims, w, om, gm, ss, forced, foff)
    assert ex == tot, f"{tot - ex} flagged near-ties"


def test_config0_tiny192_aan():
    """BASELINE configs[0]: tiny-192 AAN, 36k vocab, 4 sentences of length 20."""
    dims = synth.PRESETS["tiny192-aan"]
    w, om, gm = pair(dims, 1)
    ss = synth.uniform_set(4, 20, seed=7)
    ref = om.decode_many(ss, 4)
    got = gm.translate(ss, 8192)
    assert all(np.array_equal(a, b) for a, b in zip(got, ref))
    T = np.full(4, 20)
    foff = np.concatenate([[0], np.cumsum(T)]).astype(np.int64)
    forced = synth.forced_targets(T.tolist(), seed=9)
    tot, ex, fl = run_forced_parity(dims, w, om, gm, ss, forced, foff, layers=True)
    assert ex == tot


def test_tiny192_noffn_nogate_eos_and_edges():
    """EOS handling + compaction: with the EOS bias raised to 16 (the top logits of this
    random student are ~17-18) about half of the sentences emit EOS at step 1 (nothing is
    written, R16) and the rest run to their own max_len (0..39), so live rows drop out at
    many different steps.  Random-init students repeat one token per sentence, so EOS
    cannot be made to win mid-sentence; teacher-forced tests carry the id diversity."""
    dims = synth.PRESETS["tiny192-aan-noffn-nogate"]
    w = synth.make_weights(dims, seed=4)
    w["out.b"] = w["out.b"].copy()
    w["out.b"][dims.eos_id] = 16.0
    ss = synth.random_set(40, 0, 30, seed=8)
    ss.max_len[:] = np.random.default_rng(2).integers(0, 40, size=40)
    om, gm = O.OracleModel(dims, w), M.Model(dims, w)
    ref = om.decode_many(ss, 4)
    got = gm.translate(ss, 100)
    assert all(np.array_equal(a, b) for a, b in zip(got, ref))
    n_eos = sum(len(r) == 0 and m > 0 for r, m in zip(ref, ss.max_len))
    n_full = sum(len(r) == m > 0 for r, m in zip(ref, ss.max_len))
    assert n_eos >= 5 and n_full >= 5, (n_eos, n_full)


def test_batch_and_order_invariance():
    dims = synth.PRESETS["tiny192-aan"]
    w = synth.make_weights(dims, seed=2)
    gm = M.Model(dims, w)
    ss = synth.random_set(120, 1, 40, seed=21)
    base = gm.translate(ss, 1 << 20)
    for budget in (1, 64, 333, 4096):
        assert all(np.array_equal(a, b) for a, b in zip(gm.translate(ss, budget), base))
    for lanes in (1, 2, 3):                # concurrent decoder lanes: identical ids
        gm.set_option("lanes", lanes)
        for rows in (7, 50, 1 << 20):      # co-scheduled batch waves: identical ids
            gm.set_option("max_concurrent_rows", rows)
            assert all(np.array_equal(a, b) for a, b in zip(gm.translate(ss, 64), base))
        for tiers in (10, 30):             # length-tiered lanes (prioritised streams)
            gm.set_option("lane_tiers", tiers)
            assert all(np.array_equal(a, b) for a, b in zip(gm.translate(ss, 64), base))
            if lanes > 1:                  # critical lane in its own SM partition (green context)
                gm.set_option("green_sms", 48)
                assert all(np.array_equal(a, b) for a, b in zip(gm.translate(ss, 64), base))
                gm.set_option("green_sms", 0)
        gm.set_option("lane_tiers", 0)
    for k in (3, 8):                       # several decoder steps per CUDA graph
        gm.set_option("steps_per_graph", k)
        assert all(np.array_equal(a, b) for a, b in zip(gm.translate(ss, 333), base))
    gm.set_option("steps_per_graph", 1)
    gm.set_option("max_concurrent_rows", 0)
    gm.set_option("lanes", 1)
    perm = np.random.default_rng(3).permutation(ss.n)
    sub = gm.decode(ss.subset(perm))
    assert all(np.array_equal(sub[k], base[perm[k]]) for k in range(ss.n))


def test_errors_and_fail_fast():
    dims = ModelDims("t", 32, 64, 4, vocab=64, enc_layers=1, dec_layers=1)
    with pytest.raises(M.MnmtError) as e:
        M.Model(ModelDims("bad", 30, 64, 4))
    assert e.value.status == 1
    gm = M.Model(dims)
    with pytest.raises(M.MnmtError) as e:
        gm.set_param("enc.0.self.q.W", np.zeros(7, np.float32))
    assert e.value.status == 2
    with pytest.raises(M.MnmtError) as e:
        gm.decode(synth.uniform_set(1, 3, vocab=64))
    assert e.value.status == 4                      # before quantize
    with pytest.raises(M.MnmtError) as e:
        gm.quantize()                               # missing parameters
    assert e.value.status == 4
    gm = M.Model(dims, synth.make_weights(dims, 1))
    bad = synth.uniform_set(1, 3, vocab=64)
    bad.ids[1] = 64
    with pytest.raises(M.MnmtError) as e:
        gm.decode(bad)
    assert e.value.status == 3
    with pytest.raises(M.MnmtError) as e:
        gm.translate(synth.uniform_set(1, 3, vocab=64), 0)
    assert e.value.status == 1


# ------------------------------------------------------------------ full-size sampled parity
def _sampled(dims, n_sample, seed, budget=8192):
    w = synth.make_weights(dims, seed=1)
    gm = M.Model(dims, w)
    ss = synth.newstest_set()
    got = gm.translate(ss, budget)                  # the launch configuration bench.py times
    om = O.OracleModel(dims, w)
    L = ss.lengths
    rng = np.random.default_rng(seed)
    idx = list(rng.choice(ss.n, size=n_sample - 2, replace=False)) + [int(np.argmax(L)), int(np.argmin(L))]
    ref = om.decode_many(ss.subset(idx), 0)
    agree = sum(np.array_equal(got[i], r) for i, r in zip(idx, ref))
    words = sum(len(g) for g in got)
    return agree, len(idx), words, ss


def test_config1_small_aan_newstest_sampled():
    agree, n, words, ss = _sampled(synth.PRESETS["small-aan"], 16, 5)
    assert agree == n
    assert words <= int(ss.max_len.sum())


@pytest.mark.slow
def test_config2_base_selfattn_sampled():
    agree, n, _, _ = _sampled(synth.PRESETS["base"], 6, 6)
    assert agree == n
