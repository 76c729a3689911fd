"""P-0 pins of the oracle's beam search (
the b=2 systems of Table 3 rows 6 and 12; readings R26-R29
in DESIGN.md).

None of these re-runs the oracle's search loop: each pin is a reduction (b=1 is
greedy decoding), an exhaustive enumeration over every sequence of a toy
model whose log-probabilities come from the INDEPENDENT parallel training-time
formulation (tests/ref_parallel.py), a closed form of the log-sum-exp, or an
invariant of the n-best contract (sorted, exactly b hypotheses, scores equal to
the re-scored sequences).
"""
import itertools
import math

import numpy as np
import pytest

import synth
from synth import ModelDims
from tests import ref_parallel as RP
from tests.test_oracle_pins import tiny_variants


def lse32(row: np.ndarray) -> np.float32:
    """fl32(M + log sum exp(l - M)), written with numpy float64 (R26)."""
    z = row.astype(np.float64)
    M = z.max()
    return np.float32(M + math.log(np.exp(z - M).sum()))


def rescore(pm, src, ids, eos, finished_by_eos):
    """Score of a finished hypothesis from the parallel form's teacher-forced logits:
    sum over its steps of fl32(l_j - lse) in fp32 (R27); an EOS-finished hypothesis
    also pays log p(EOS) at its last step."""
    T = len(ids) + (1 if finished_by_eos else 0)
    forced = np.array(list(ids) + [0], np.int32)
    _, _, logits = pm.forced(src, forced, T)
    s = np.float32(0.0)
    for t in range(T):
        tok = ids[t] if t < len(ids) else eos
        s = np.float32(s + np.float32(logits[t, tok] - lse32(logits[t])))
    return s


def test_logsumexp_closed_forms(orc):
    V = 36000
    for c in (0.0, -3.25, 17.5):
        l = np.full(V, c, np.float32)
        assert orc.logsumexp(l) == np.float32(c + math.log(V))
    # one dominant logit: lse -> that logit; softmax of the others underflows in fp32
    l = np.full(100, -200.0, np.float32); l[7] = 5.0
    assert orc.logsumexp(l) == np.float32(5.0)
    # probabilities from the fp32 log-softmax sum to 1 within V fp32 roundings
    rng = np.random.default_rng(0)
    l = rng.normal(0, 3, 5000).astype(np.float32)
    lp = l - np.float32(orc.logsumexp(l))
    assert abs(np.exp(lp.astype(np.float64)).sum() - 1.0) < 5000 * 2 ** -23


@pytest.fixture(scope="module")
def varied_models(orc):
    """Tiny students with a small embedding scale, so free-running outputs vary."""
    out = []
    for i, m in enumerate(tiny_variants()):
        w = synth.make_weights(m, seed=200 + i, emb_scale=0.05)
        out.append((m, w, orc.OracleModel(m, w), RP.ParallelModel(m, w)))
    return out


def test_beam1_equals_greedy(varied_models):
    """b = 1 reduces to greedy decoding, token for token."""
    for m, w, om, pm in varied_models:
        ss = synth.random_set(6, 1, 12, seed=51, vocab=m.vocab)
        for i in range(ss.n):
            src = ss.ids[ss.offsets[i]:ss.offsets[i + 1]]
            g = om.decode_one(src, 9)
            nb = om.beam_one(src, 9, 1)
            assert len(nb) == 1
            assert nb[0][0].tolist() == g.tolist(), m.name


def test_beam_nbest_contract_and_rescoring(varied_models):
    """Exactly b hypotheses, sorted by descending score; every score equals the sum of
    fp32 log-probabilities of its ids under the parallel (training-time) formulation —
    this checks that each hypothesis carried the decoder state of its own prefix."""
    for m, w, om, pm in varied_models:
        ss = synth.random_set(3, 2, 9, seed=61, vocab=m.vocab)
        for b in (2, 3, 5):
            for i in range(ss.n):
                src = ss.ids[ss.offsets[i]:ss.offsets[i + 1]]
                T = 6
                nb = om.beam_one(src, T, b)
                assert len(nb) == b, m.name
                scores = [s for _, s in nb]
                assert all(scores[k] >= scores[k + 1] for k in range(b - 1)), m.name
                for ids, s in nb:
                    assert len(ids) <= T
                    assert m.eos_id not in ids.tolist()
                    by_eos = len(ids) < T
                    r = rescore(pm, src, ids.tolist(), m.eos_id, by_eos)
                    assert abs(float(r) - s) <= 1e-5 * max(1.0, abs(s)), (m.name, ids, s, r)


TOY = ModelDims("toy", 16, 32, 2, vocab=6, enc_layers=1, dec_layers=1)


@pytest.mark.parametrize("decoder", [1, 0])
def test_beam_equals_exhaustive_enumeration(orc, decoder):
    """b = |V| on a 2-step toy model: the beam's n-best list equals the exhaustive
    enumeration of every sequence (S:L458 'top hypothesis equals exhaustive enumeration
    argmax'; here the whole list): step 1 keeps all |V| candidates (the EOS one finishes),
    step 2 = max_len keeps the |V|-1 best two-step sequences."""
    m = ModelDims("toy", 16, 32, 2, vocab=6, enc_layers=1, dec_layers=1, decoder=decoder)
    V, eos = m.vocab, m.eos_id
    for seed in range(3):
        w = synth.make_weights(m, seed=300 + seed, emb_scale=0.3)
        om, pm = orc.OracleModel(m, w), RP.ParallelModel(m, w)
        src = np.array([3, 4, 5, 1][: 2 + seed], np.int32)
        _, _, l1 = pm.forced(src, np.zeros(1, np.int32), 1)
        lp1 = (l1[0] - lse32(l1[0])).astype(np.float32)
        seqs = [((), np.float32(0.0) + lp1[eos], 0, eos, float(l1[0, eos]))]
        two = []
        for s1 in range(V):
            if s1 == eos:
                continue
            _, _, l2 = pm.forced(src, np.array([s1, 0], np.int32), 2)
            lp2 = (l2[1] - lse32(l2[1])).astype(np.float32)
            for s2 in range(V):
                sc = np.float32(np.float32(0.0 + lp1[s1]) + lp2[s2])
                ids = (s1,) if s2 == eos else (s1, s2)
                two.append((ids, sc, s1, s2, float(l2[1, s2])))
        # all scores distinct: the tie-break order (R28) does not matter here
        all_sc = [float(x[1]) for x in two] + [float(seqs[0][1])]
        assert len(set(all_sc)) == len(all_sc)
        two.sort(key=lambda x: -float(x[1]))
        expect = sorted(seqs + two[: V - 1], key=lambda x: -float(x[1]))
        nb = om.beam_one(src, 2, V)
        assert [tuple(i.tolist()) for i, _ in nb] == [e[0] for e in expect]
        assert np.allclose([s for _, s in nb], [float(e[1]) for e in expect], rtol=0, atol=1e-6)
        # and the top hypothesis is the argmax over ALL sequences of length <= 2
        best = max(seqs + two, key=lambda x: float(x[1]))
        assert tuple(nb[0][0].tolist()) == best[0]


def test_beam_ties_follow_rank_order(orc):
    """Equal logits everywhere (E = 0, no bias): every candidate scores the same, so the
    order R28 decides: logit (equal), hypothesis rank, then lowest id.  With b = 3 the kept
    step-1 candidates are ids 0 (EOS, finished), 1, 2; step 2 expands hypothesis [1] first."""
    m = ModelDims("toy", 16, 32, 2, vocab=6, enc_layers=1, dec_layers=1, out_bias=0)
    w = synth.make_weights(m, seed=5)
    w["emb.E"] = np.zeros_like(w["emb.E"])
    om = orc.OracleModel(m, w)
    nb = om.beam_one(np.array([3, 4], np.int32), 2, 3)
    assert [i.tolist() for i, _ in nb] == [[], [1], [1, 1]]
    lp = np.float32(-np.float32(math.log(6)))
    assert [s for _, s in nb] == [lp, np.float32(lp + lp), np.float32(lp + lp)]


def test_beam_edge_cases(orc):
    m = TOY
    om = orc.OracleModel(m, synth.make_weights(m, seed=9))
    assert om.beam_one(np.array([3], np.int32), 0, 2) == []          # max_len 0
    nb = om.beam_one(np.zeros(0, np.int32), 3, 2)                     # empty source
    assert len(nb) == 2
    with pytest.raises(ValueError):
        om.beam_one(np.array([3], np.int32), 3, 0)                    # b < 1
    with pytest.raises(ValueError):
        om.beam_one(np.array([3], np.int32), 3, m.vocab + 1)          # b > |V|
    # EOS always first: every hypothesis finishes at step 1 with the empty sequence ... and
    # the other b-1 kept candidates at step 1 continue; EOS-biased model -> all finish by EOS
    w = synth.make_weights(m, seed=9); w["out.b"] = w["out.b"].copy(); w["out.b"][0] = 50.0
    om2 = orc.OracleModel(m, w)
    nb = om2.beam_one(np.array([3, 4], np.int32), 5, 2)
    assert nb[0][0].tolist() == [] and len(nb) == 2


def test_beam_many_matches_beam_one(varied_models):
    m, w, om, pm = varied_models[0]
    ss = synth.random_set(5, 1, 10, seed=71, vocab=m.vocab)
    many = om.beam_many(ss, 3)
    for i in range(ss.n):
        src = ss.ids[ss.offsets[i]:ss.offsets[i + 1]]
        one = om.beam_one(src, int(ss.max_len[i]), 3)
        assert [(a.tolist(), s) for a, s in many[i]] == [(a.tolist(), s) for a, s in one]
