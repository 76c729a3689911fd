"""Beam search: libmnmt's mnmt_beam_translate against the oracle's
orc_beam_one (tests/test_oracle_beam.py pins the oracle).

Bar: for every sentence the n-best list (ids, lengths, count) is identical to the oracle's and
every score is the oracle's fp32 score (bit-exact in practice: the only float difference is
the fp64 order of the log-sum-exp, R26, which moves the fp32 lse only on a rounding-boundary
straddle).  b = 1 must reproduce greedy decoding.
"""
import numpy as np
import pytest

import oracle.oracle as O
import synth
from synth import ModelDims

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1805_12096_b200 import mnmt as M  # noqa: E402

VARIANTS = [
    ModelDims("t-aan", 32, 64, 4, vocab=64, enc_layers=2, dec_layers=2),
    ModelDims("t-ffn1", 32, 64, 4, vocab=64, enc_layers=2, dec_layers=2, aan_ffn_depth=1),
    ModelDims("t-noffn-nogate", 32, 64, 4, vocab=64, enc_layers=2, dec_layers=2,
              aan_ffn_depth=0, aan_gate=0),
    ModelDims("t-self", 32, 64, 4, vocab=64, enc_layers=2, dec_layers=2, decoder=0),
    ModelDims("t-nobias-ragged-vocab", 48, 96, 4, vocab=50, enc_layers=1, dec_layers=3, out_bias=0),
    ModelDims("t192-aan-v1000", 192, 384, 8, vocab=1000, enc_layers=2, dec_layers=2),
    ModelDims("t256-self-v1000", 256, 512, 8, vocab=1000, enc_layers=2, dec_layers=2, decoder=0),
]


def pair(dims, seed, emb_scale=0.05):
    w = synth.make_weights(dims, seed=seed, emb_scale=emb_scale)
    return w, O.OracleModel(dims, w), M.Model(dims, w)


def compare(got, ref, tag):
    """Identical n-best lists; scores equal up to an fp32 lse rounding-boundary event."""
    n_sc, n_exact = 0, 0
    for i, (g, r) in enumerate(zip(got, ref)):
        assert len(g) == len(r), (tag, i, len(g), len(r))
        for (gi, gs), (ri, rs) in zip(g, r):
            assert np.array_equal(gi, ri), (tag, i, gi, ri)
            assert abs(gs - rs) <= 1e-5 * max(1.0, abs(rs)), (tag, i, gs, rs)
            n_sc += 1
            n_exact += gs == rs
    assert n_exact >= 0.99 * n_sc, (tag, n_exact, n_sc)
    return n_sc


@pytest.mark.parametrize("dims", VARIANTS, ids=lambda d: d.name)
@pytest.mark.parametrize("beam", [2, 4])
def test_beam_matches_oracle(dims, beam):
    w, om, gm = pair(dims, 31)
    ss = synth.random_set(23, 1, 14, seed=9, vocab=dims.vocab)
    ref = om.beam_many(ss, beam, 4)
    for fused in (0, 1):   # logits + row reduction, or log-sum-exp / top-k in the GEMM epilogue
        gm.set_option("beam_fused", fused)
        got = gm.beam_translate(ss, 40, beam)
        assert compare(got, ref, f"{dims.name} fused={fused}") == beam * ss.n


@pytest.mark.parametrize("dims", VARIANTS[:4], ids=lambda d: d.name)
def test_beam1_is_greedy(dims):
    w, om, gm = pair(dims, 32)
    ss = synth.random_set(19, 1, 12, seed=10, vocab=dims.vocab)
    greedy = gm.translate(ss, 64)
    nb = gm.beam_translate(ss, 64, 1)
    assert all(len(h) == 1 and np.array_equal(h[0][0], g) for h, g in zip(nb, greedy))
    compare(nb, om.beam_many(ss, 1, 4), dims.name)


def test_beam8_and_edges():
    """b = 8 (the TOPK limit), empty sources, max_len 0 (no hypotheses), max_len 1, and an
    EOS-biased output layer so that hypotheses finish at many different steps."""
    dims = ModelDims("t-aan-v300", 64, 128, 4, vocab=300, enc_layers=2, dec_layers=2)
    w = synth.make_weights(dims, seed=33, emb_scale=0.05)
    w["out.b"] = w["out.b"].copy()
    w["out.b"][dims.eos_id] = 2.5
    om, gm = O.OracleModel(dims, w), M.Model(dims, w)
    ss = synth.random_set(30, 0, 20, seed=11, vocab=dims.vocab)
    ss.max_len[:] = np.random.default_rng(4).integers(0, 12, size=ss.n)
    ss.max_len[:3] = [0, 1, 2]
    for beam, fused in ((3, 0), (8, 0), (8, 1)):
        gm.set_option("beam_fused", fused)
        ref = om.beam_many(ss, beam, 4)
        got = gm.beam_translate(ss, 25, beam)
        compare(got, ref, f"b{beam}")
        assert all(len(g) == (beam if m > 0 else 0) for g, m in zip(got, ss.max_len))
        lens = [len(h[0]) for g in got for h in g]
        assert min(lens) < max(lens)   # hypotheses ended at different steps


def test_beam_invariance_over_scheduling():
    """Ids and scores do not depend on batching, lanes, tiers or SM partitions."""
    dims = ModelDims("t192-aan", 192, 384, 8, vocab=1000, enc_layers=2, dec_layers=2)
    w, om, gm = pair(dims, 34)
    ss = synth.random_set(90, 1, 30, seed=12, vocab=dims.vocab)
    base = gm.beam_translate(ss, 1 << 20, 2)
    compare(base, om.beam_many(ss, 2, 0), "ref")
    for budget in (1, 77, 500):
        got = gm.beam_translate(ss, budget, 2)
        assert all([(a.tolist(), s) for a, s in x] == [(a.tolist(), s) for a, s in y]
                   for x, y in zip(got, base)), budget
    gm.set_option("lanes", 3)
    gm.set_option("lane_tiers", 40)
    gm.set_option("max_concurrent_rows", 4096)
    gm.set_option("green_sms", 48)
    got = gm.beam_translate(ss, 64, 2)
    assert all([(a.tolist(), s) for a, s in x] == [(a.tolist(), s) for a, s in y]
               for x, y in zip(got, base))
    # greedy after beam on the same handle is unaffected
    assert all(np.array_equal(a, b) for a, b in zip(gm.translate(ss, 64), om.decode_many(ss, 0)))


def test_beam_small_aan_36k_vocab():
    """configs[1] dims (small AAN, V = 36000: 282 TOPK partials per row), b = 2 and 4."""
    dims = synth.PRESETS["small-aan"]
    w, om, gm = pair(dims, 1, emb_scale=0.5)
    ss = synth.random_set(6, 3, 16, seed=13)
    for beam in (2, 4):
        ref = om.beam_many(ss, beam, 0)
        for fused in (0, 1):
            gm.set_option("beam_fused", fused)
            compare(gm.beam_translate(ss, 8192, beam), ref, f"small b{beam} fused={fused}")


def test_beam_errors():
    dims = VARIANTS[0]
    w, om, gm = pair(dims, 35)
    ss = synth.random_set(3, 1, 5, seed=14, vocab=dims.vocab)
    for bad in (0, 9):
        with pytest.raises(M.MnmtError):
            gm.beam_translate(ss, 10, bad)
