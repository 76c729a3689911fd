"""Vocabulary shortlist: libmnmt's mnmt_translate with
MNMT_SHORTLIST against the oracle (orc_build_shortlist + orc_decode_many_sl per word-budget
batch; tests/test_oracle_shortlist.py and tests/test_golden.py pin the oracle).

Bar: token ids bit-exact for every sentence (integer union, integer GEMM accumulators, the same
fp32 logits over the shortlisted columns; the lowest id wins ties since the shortlist is
ascending, R15/R33).
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
    (ModelDims("t-aan", 32, 64, 4, vocab=64, enc_layers=2, dec_layers=2), 4, 3),
    (ModelDims("t-self", 32, 64, 4, vocab=64, enc_layers=2, dec_layers=2, decoder=0), 4, 3),
    (ModelDims("t-nobias-ragged-vocab", 48, 96, 4, vocab=50, enc_layers=1, dec_layers=3,
               out_bias=0), 3, 2),
    (ModelDims("t192-aan-v1000", 192, 384, 8, vocab=1000, enc_layers=2, dec_layers=2), 40, 12),
    (ModelDims("t256-self-v3000", 256, 512, 8, vocab=3000, enc_layers=2, dec_layers=2,
               decoder=0), 100, 25),
]


def oracle_shortlist_job(om, dims, sset, budget, freq, lex):
    """The paper's procedure on the CPU: sorted word-budget batches, each decoded over
    the union of the frequent list and its source words' translations."""
    order, off = O.batch_by_words(sset.lengths, budget)
    res = [None] * sset.n
    sizes = []
    for b in range(len(off) - 1):
        idx = order[off[b]:off[b + 1]]
        sub = sset.subset(idx)
        sl = O.build_shortlist(dims.vocab, freq, lex, sub.ids, eos=dims.eos_id, unk=1)
        sizes.append(sl.size)
        for i, ids in zip(idx, om.decode_many_sl(sub, sl, 4)):
            res[i] = ids
    return res, sizes


def check(got, ref, tag):
    for i, (g, r) in enumerate(zip(got, ref)):
        assert np.array_equal(g, r), (tag, i, g, r)


@pytest.mark.parametrize("dims,n_freq,k_lex", VARIANTS, ids=lambda v: getattr(v, "name", str(v)))
@pytest.mark.parametrize("budget", [1, 40, 10_000])
def test_shortlist_matches_oracle(dims, n_freq, k_lex, budget):
    w = synth.make_weights(dims, seed=41, emb_scale=0.05)
    om, gm = O.OracleModel(dims, w), M.Model(dims, w)
    freq, lex = synth.shortlist_tables(dims.vocab, n_freq, k_lex, seed=8)
    gm.set_shortlist(freq, lex)
    ss = synth.random_set(29, 1, 17, seed=12, vocab=dims.vocab)
    ref, sizes = oracle_shortlist_job(om, dims, ss, budget, freq, lex)
    assert min(sizes) < dims.vocab          # the restriction is real
    check(gm.translate(ss, budget, shortlist=True), ref, (dims.name, budget))
    allowed = set(freq.tolist()) | set(lex[ss.ids].ravel().tolist()) | {0, 1}
    for g in gm.translate(ss, budget, shortlist=True):
        assert set(g.tolist()) <= allowed


def test_shortlist_scheduling_options():
    """Tiered lanes, green contexts, co-scheduled waves and the persistent step kernel option
    (bypassed) change no id."""
    dims = ModelDims("t192-aan-v1000", 192, 384, 8, vocab=1000, enc_layers=2, dec_layers=2)
    w = synth.make_weights(dims, seed=42, emb_scale=0.05)
    om, gm = O.OracleModel(dims, w), M.Model(dims, w)
    freq, lex = synth.shortlist_tables(dims.vocab, 30, 10, seed=9)
    gm.set_shortlist(freq, lex)
    ss = synth.random_set(60, 1, 40, seed=13, vocab=dims.vocab)
    ref, _ = oracle_shortlist_job(om, dims, ss, 120, freq, lex)
    check(gm.translate(ss, 120, shortlist=True), ref, "default")
    for name, v in [("lanes", 3), ("lane_tiers", 40), ("max_concurrent_rows", 4096),
                    ("green_sms", 48), ("pers_reserve", 16)]:
        gm.set_option(name, v)
    check(gm.translate(ss, 120, shortlist=True), ref, "bench options")
    # a plain call after shortlisted ones is the unrestricted decode again
    check(gm.translate(ss, 120), om.decode_many(ss, 4), "plain after shortlist")


@pytest.mark.parametrize("budget", [1, 25, 300])
def test_shortlist_co_scheduled_waves(budget):
    """Many word-budget batches per decode wave (budget 1: one sentence per batch, 150 batches,
    so waves hit the 64-group cap): one output GEMM over the wave's union, every row masked to
    its own batch's shortlist."""
    dims = ModelDims("t192-aan-v1000", 192, 384, 8, vocab=1000, enc_layers=2, dec_layers=2)
    w = synth.make_weights(dims, seed=45, emb_scale=0.05)
    om, gm = O.OracleModel(dims, w), M.Model(dims, w)
    freq, lex = synth.shortlist_tables(dims.vocab, 20, 8, seed=11)
    gm.set_shortlist(freq, lex)
    ss = synth.random_set(150, 1, 30, seed=16, vocab=dims.vocab)
    ref, _ = oracle_shortlist_job(om, dims, ss, budget, freq, lex)
    gm.set_option("max_concurrent_rows", 4096)
    check(gm.translate(ss, budget, shortlist=True), ref, ("waves", budget))
    gm.set_option("lanes", 3)
    gm.set_option("lane_tiers", 40)
    check(gm.translate(ss, budget, shortlist=True), ref, ("waves+tiers", budget))


def test_full_vocabulary_shortlist_is_plain_greedy():
    dims = ModelDims("t-aan", 32, 64, 4, vocab=64, enc_layers=2, dec_layers=2)
    w = synth.make_weights(dims, seed=43, emb_scale=0.05)
    gm = M.Model(dims, w)
    gm.set_shortlist(np.arange(dims.vocab, dtype=np.int32), np.zeros((dims.vocab, 0), np.int32))
    ss = synth.random_set(17, 1, 12, seed=14, vocab=dims.vocab)
    check(gm.translate(ss, 30, shortlist=True), gm.translate(ss, 30), "full")


def test_padding_entries_and_errors():
    dims = ModelDims("t-aan", 32, 64, 4, vocab=64, enc_layers=2, dec_layers=2)
    w = synth.make_weights(dims, seed=44, emb_scale=0.05)
    om, gm = O.OracleModel(dims, w), M.Model(dims, w)
    ss = synth.random_set(9, 1, 10, seed=15, vocab=dims.vocab)
    with pytest.raises(M.MnmtError):
        gm.translate(ss, 30, shortlist=True)              # no tables yet: MNMT_ERR_STATE
    freq, lex = synth.shortlist_tables(dims.vocab, 4, 4, seed=10)
    lex[:, -1] = -1                                       # padding entries are ignored
    lex[::3, 0] = dims.vocab + 7
    gm.set_shortlist(freq, lex)
    ref, _ = oracle_shortlist_job(om, dims, ss, 30, freq, lex)
    check(gm.translate(ss, 30, shortlist=True), ref, "padded")
    assert M.lib().mnmt_model_set_shortlist(gm.h, None, -1, None, 0) == 1   # MNMT_ERR_ARG


def test_tiny192_newstest_slice_full_vocab():
    """configs[0] model (36k vocabulary) with the paper's 100 + 100 tables."""
    dims = synth.PRESETS["tiny192-aan"]
    w = synth.make_weights(dims, seed=1)
    om, gm = O.OracleModel(dims, w), M.Model(dims, w)
    freq, lex = synth.shortlist_tables(dims.vocab, 100, 100, seed=85)
    gm.set_shortlist(freq, lex)
    ss = synth.newstest_set().subset(np.arange(0, 3003, 150))
    ref, sizes = oracle_shortlist_job(om, dims, ss, 96, freq, lex)
    assert max(sizes) < dims.vocab // 4
    check(gm.translate(ss, 96, shortlist=True), ref, "tiny192")
