"""P-0 pins of the oracle's vocabulary shortlist ("the union of
the 100 most frequent target words and the 100 most probable translations for every source word
in a batch").

Pins: SPEC's examples (vocabulary smaller than the frequent list -> whole vocabulary; shared
translations deduplicated), a brute-force Python set union on random tables, and decoding:
the full-vocabulary shortlist reduces to plain greedy decoding, and a restricted decode equals
the brute-force argmax over the shortlisted logits of the independent parallel formulation.
"""
import numpy as np

import synth
from synth import ModelDims
from tests import ref_parallel as RP


def test_spec_examples(orc):
    V = 50
    freq = np.arange(V, dtype=np.int32)[::-1].copy()            # all 50 words are "frequent"
    lex = np.zeros((V, 3), np.int32)
    assert orc.build_shortlist(V, freq, lex, np.array([3, 4], np.int32)).tolist() == list(range(V))
    # two source tokens sharing translations: the union is deduplicated (set semantics)
    V = 1000
    lex = np.full((V, 3), 999, np.int32)
    lex[10] = [500, 600, 700]
    lex[11] = [600, 700, 800]
    sl = orc.build_shortlist(V, np.array([], np.int32), lex, np.array([10, 11, 10], np.int32))
    assert sl.tolist() == [0, 1, 500, 600, 700, 800]            # + EOS (0) and UNK (1)


def test_matches_bruteforce_union(orc):
    rng = np.random.default_rng(0)
    for _ in range(20):
        V = int(rng.integers(20, 3000))
        k = int(rng.integers(1, 12))
        lex = rng.integers(0, V, size=(V, k)).astype(np.int32)
        freq = rng.choice(V, size=min(V, int(rng.integers(0, 120))), replace=False).astype(np.int32)
        src = rng.integers(0, V, size=int(rng.integers(0, 60))).astype(np.int32)
        got = orc.build_shortlist(V, freq, lex, src, eos=0, unk=1)
        want = sorted(set(freq.tolist()) | {int(j) for s in src for j in lex[s]} | {0, 1})
        assert got.tolist() == want


def test_full_shortlist_is_plain_greedy(orc):
    m = ModelDims("t", 32, 64, 4, vocab=64, enc_layers=2, dec_layers=2)
    w = synth.make_weights(m, seed=21, emb_scale=0.05)
    om = orc.OracleModel(m, w)
    ss = synth.random_set(7, 1, 12, seed=3, vocab=m.vocab)
    full = om.decode_many_sl(ss, np.arange(m.vocab, dtype=np.int32), 2)
    assert all(np.array_equal(a, b) for a, b in zip(full, om.decode_many(ss, 2)))


def test_restricted_decode_equals_bruteforce(orc):
    """Each step's id = the highest shortlisted logit (lowest id on ties) of the parallel form run
    on the prefix decoded so far; every emitted id is in the shortlist."""
    for dec in (1, 0):
        m = ModelDims("t", 32, 64, 4, vocab=64, enc_layers=2, dec_layers=2, decoder=dec)
        w = synth.make_weights(m, seed=22, emb_scale=0.05)
        om, pm = orc.OracleModel(m, w), RP.ParallelModel(m, w)
        rng = np.random.default_rng(4)
        sl = np.sort(rng.choice(np.arange(2, m.vocab), size=15, replace=False)).astype(np.int32)
        sl = np.concatenate([[0], sl]).astype(np.int32)            # EOS included
        ss = synth.random_set(4, 2, 9, seed=5, vocab=m.vocab)
        got = om.decode_many_sl(ss, sl, 1)
        for i in range(ss.n):
            src = ss.ids[ss.offsets[i]:ss.offsets[i + 1]]
            prefix = []
            for t in range(1, int(ss.max_len[i]) + 1):
                _, _, lg = pm.forced(src, np.array(prefix + [0], np.int32), t)
                nxt = int(sl[np.argmax(lg[t - 1][sl])])
                if nxt == m.eos_id:
                    break
                prefix.append(nxt)
            assert got[i].tolist() == prefix
            assert set(got[i].tolist()) <= set(sl.tolist())
