"""P-0 pins of the oracle's paper-faithful CPU arithmetic variants (oracle
only, no GPU kernel): int8 codes with saturating int16 accumulation of adjacent pairs
("We accumulated in 16-bit integers with saturation"), and int16 codes x 2^10
 with wrapping 32-bit accumulation ("there is no AVX512F instruction for 32-bit
add with saturation").  The GPU path is the exact-s32 arithmetic (R3); these variants only
quantify how far the paper's CPU numerics depart from it (scripts/arith_departure.py).

Pins: SPEC.md's worked examples, hand-computed saturation / wrap-around values,
equality with the exact sum wherever no saturation or overflow can occur (brute force), and a
whole-decoder reduction (a model whose accumulators provably never leave int16 decodes
identically under saturating and exact accumulation).
"""
import numpy as np
import pytest

import synth
from synth import ModelDims


def test_q16_spec_examples(orc):
    assert [orc.q16(x) for x in (1.0, 0.0, -0.5)] == [1024, 0, -512]
    assert orc.q16(40.0) == 32767 and orc.q16(-40.0) == -32767            # S:L117 (saturated)
    xs = np.random.default_rng(0).uniform(-16, 16, 2000).astype(np.float32)
    err = np.abs(np.array([orc.q16(x) for x in xs]) / 1024.0 - xs.astype(np.float64))
    assert err.max() <= 2.0 ** -11                                         # S:L118 half step
    # ties round to even (R1): 0.5/1024 and 1.5/1024 are exact halves
    assert orc.q16(0.5 / 1024) == 0 and orc.q16(1.5 / 1024) == 2 and orc.q16(-2.5 / 1024) == -2


def test_int16_product_spec_example(orc):
    a = [orc.q16(1.0), orc.q16(2.0)]
    w = [orc.q16(0.5), orc.q16(0.25)]
    acc = orc.dot_codes(orc.ARITH_INT16, a, w)
    assert acc == 1 << 20                       # 1024*512 + 2048*256 = 2^20
    assert acc / 2.0 ** 20 == 1.0


def test_int16_wraps_at_32_bits(orc):
    a = [32767] * 3
    assert orc.dot_codes(orc.ARITH_INT16, a, a) == 3 * 32767 * 32767 - (1 << 32)   # -1073938429
    assert orc.dot_codes(orc.ARITH_S32, [100] * 3, [100] * 3) == 30000


def test_sat16_spec_examples(orc):
    assert orc.dot_codes(orc.ARITH_SAT16, [64], [64]) == 4096                     # S:L144 (odd K padded)
    assert orc.dot_codes(orc.ARITH_SAT16, [127] * 16, [127] * 16) == 32767         # S:L146 pinned
    assert orc.dot_codes(orc.ARITH_SAT16, [127] * 16, [-127] * 16) == -32768       # lower rail
    # pair sums of 2*127*127 = 32258 fit in int16 and cancel exactly
    assert orc.dot_codes(orc.ARITH_SAT16, [127, 127, 127, 127], [127, 127, -127, -127]) == 0
    # saturation is not undone by later terms of the other sign (sequential, not exact)
    assert orc.dot_codes(orc.ARITH_SAT16, [127] * 6 + [-127] * 2, [127] * 8) == 32767 - 32258


@pytest.mark.parametrize("arith", [1, 2])
def test_variants_equal_exact_sum_without_saturation(orc, arith):
    """with inputs bounded so that nothing saturates / overflows, the variants equal the
    exact sum (brute force over random vectors)."""
    rng = np.random.default_rng(arith)
    for K in (1, 2, 7, 8, 64):
        for _ in range(50):
            bound = 11 if arith == 1 else 127
            a = rng.integers(-bound, bound + 1, K)
            w = rng.integers(-bound, bound + 1, K)
            if arith == 1 and K * bound * bound > 32767:
                continue
            assert orc.dot_codes(arith, a, w) == int(np.dot(a.astype(np.int64), w.astype(np.int64)))


def test_sat16_decoder_equals_exact_when_accumulators_fit(orc):
    """Whole-decoder reduction: every weight code is in {-1, 0, 1} and every activation code is in
    [-127, 127], so with d = 16 and F = 32 every pair sum is <= 254 and every accumulator
    <= 16 * 254 < 32767: saturating int16 accumulation never triggers, and the decoder must
    produce the exact-s32 decoder's ids and outputs bit for bit."""
    m = ModelDims("toy", 16, 32, 2, vocab=40, enc_layers=1, dec_layers=2)
    rng = np.random.default_rng(7)
    w = synth.make_weights(m, seed=8)
    for k, v in w.items():
        if k.endswith(".W") or k == "emb.E":
            w[k] = (rng.integers(-1, 2, v.shape) / np.float32(63.5)).astype(np.float32)
    ex = orc.OracleModel(m, w, arith=orc.ARITH_S32)
    sa = orc.OracleModel(m, w, arith=orc.ARITH_SAT16)
    src = np.array([3, 9, 27, 5], np.int32)
    forced = synth.forced_targets([8], seed=3, vocab=m.vocab)
    i1, t1 = ex.decode_one(src, 8, forced=forced, trace=True)
    i2, t2 = sa.decode_one(src, 8, forced=forced, trace=True)
    assert np.array_equal(i1, i2)
    assert np.array_equal(t1["dec_out"], t2["dec_out"])


def test_variant_decoders_run_and_differ_from_exact(orc):
    """The variants are whole decoders (same readings otherwise); on a Table-1-shaped tiny
    student the int16 x 2^10 variant overflows its 32-bit accumulators somewhere (P:L92
    'we see overflow for the large Transformer model') or not — either way its ids are a valid
    decode; the decode is deterministic."""
    m = ModelDims("t", 64, 256, 4, vocab=300, enc_layers=2, dec_layers=2)
    w = synth.make_weights(m, seed=9, emb_scale=0.05)
    ss = synth.random_set(4, 3, 10, seed=4, vocab=m.vocab)
    for arith in (0, 1, 2):
        om = orc.OracleModel(m, w, arith=arith)
        a = om.decode_many(ss, 2)
        b = om.decode_many(ss, 1)
        assert all(np.array_equal(x, y) for x, y in zip(a, b))
        assert all(((x >= 0) & (x < m.vocab)).all() for x in a)
