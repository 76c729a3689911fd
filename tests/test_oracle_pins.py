"""P-0: pins of the CPU oracle against what the paper and mathematics fix
(SURVEY.md 8(c).3).  None of these re-types the oracle's formula: each one is a
worked example, a closed form, an invariant, a textbook special case, or an
independent formulation (tests/ref_parallel.py: parallel training-time form).
"""
import math

import numpy as np
import pytest

import synth
from synth import ModelDims
from tests import ref_parallel as RP

TINY = ModelDims("tiny-test", 32, 64, 4, vocab=64, enc_layers=2, dec_layers=2)


def tiny_variants():
    return [
        TINY,
        ModelDims("t-ffn1", 32, 64, 4, vocab=64, enc_layers=2, dec_layers=2, aan_ffn_depth=1),
        ModelDims("t-noffn-nogate", 32, 64, 4, vocab=64, enc_layers=2, dec_layers=2,
                  aan_ffn_depth=0, aan_gate=0),
        ModelDims("t-self", 32, 64, 4, vocab=64, enc_layers=2, dec_layers=2, decoder=0),
        ModelDims("t-nobias", 24, 48, 3, vocab=50, enc_layers=1, dec_layers=3, out_bias=0),
        ModelDims("t-kvbf16", 32, 64, 4, vocab=64, enc_layers=2, dec_layers=2, kv_bf16=1),
        ModelDims("t-self-kvbf16", 32, 64, 4, vocab=64, enc_layers=2, dec_layers=2, decoder=0,
                  kv_bf16=1),
    ]


# --------------------------------------------------------------- quantizer
def test_quant_spec_worked_examples(orc):
    # SPEC.md:L126-128 worked examples, c = 2 (all consistent with RNE: 63.5 -> 64 is even).
    assert orc.quantize(np.array([2.5], np.float32))[0] == 127
    assert orc.quantize(np.array([1.0], np.float32))[0] == 64
    assert list(orc.quantize(np.array([-2.0, 0.0], np.float32))) == [-127, 0]
    assert orc.sigma(2.0) == 63.5
    # s = fl32(c^2/127^2) is one float however it is formed (SURVEY 8 "Symbols").
    s = orc.dequant_scale(2.0)
    assert s == np.float32(4.0 / 16129.0) == np.float32((2.0 / 127.0) ** 2) == np.float32(1 / 63.5 ** 2)


def test_quant_round_half_even(orc):
    """Exact k+1/2 products round to the even code (R1)."""
    found = 0
    for k in range(0, 127):
        x0 = np.float32((k + 0.5) / 63.5)
        for j in range(-8, 9):
            x = x0
            for _ in range(abs(j)):
                x = np.nextafter(x, np.float32(np.inf if j > 0 else -np.inf), dtype=np.float32)
            if np.float32(x) * np.float32(63.5) == np.float32(k + 0.5):
                even = k if k % 2 == 0 else k + 1
                assert orc.quantize(np.array([x], np.float32))[0] == even
                assert orc.quantize(np.array([-x], np.float32))[0] == -even
                found += 1
    assert found >= 100    # SURVEY 8(c).2 Q1 found 129 such inputs
    # the SURVEY's example: x = fl32(5/127) -> 2 (half-away-from-zero would give 3)
    assert orc.quantize(np.array([np.float32(5 / 127)], np.float32))[0] == 2


def test_quant_code_domain_roundtrip(orc):
    k = np.arange(-127, 128)
    w = (k.astype(np.float32) / np.float32(63.5)).astype(np.float32)
    assert np.array_equal(orc.quantize(w).astype(np.int64), k)


def test_quant_error_bound_and_range(orc):
    x = synth.uniform_activations((200000,), seed=9, scale=5.0)
    q = orc.quantize(x).astype(np.float64)
    assert q.min() >= -127 and q.max() <= 127          # -128 never produced
    err = np.abs(q / 63.5 - np.clip(x.astype(np.float64), -2, 2))
    assert err.max() <= 1.0 / 127.0 + 1e-6              # half-step bound (SPEC.md:L159 form)
    xs = np.sort(x)
    assert np.all(np.diff(orc.quantize(xs).astype(np.int64)) >= 0)   # monotone


# --------------------------------------------------------------- integer product
@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (3, 5, 7), (17, 33, 130), (64, 9, 300)])
def test_gemm_bruteforce(orc, M, N, K):
    rng = np.random.default_rng(M * 1000 + N + K)
    a = rng.integers(-127, 128, size=(M, K)).astype(np.int8)
    w = rng.integers(-127, 128, size=(N, K)).astype(np.int8)
    ref = a.astype(np.int64) @ w.astype(np.int64).T       # brute force, exact
    assert np.array_equal(orc.gemm_acc(a, w).astype(np.int64), ref)


def test_gemm_spec_example(orc):
    # 1.0 -> 64; 64*64*(2/127)^2.  The SPEC prints ~1.01587; the exact
    # value is 16384/16129 = 1.015810... (the SPEC's last digits are a rounding slip).
    qa = orc.quantize(np.array([[1.0, 0.0]], np.float32))
    acc = orc.gemm_acc(qa, qa)
    assert acc[0, 0] == 4096
    assert abs(float(acc[0, 0]) * orc.dequant_scale() - 16384 / 16129) < 1e-6
    assert abs(float(acc[0, 0]) * orc.dequant_scale() - 1.01587) < 1e-4


def test_quantized_vs_float_bound(orc):
    """|s*acc - sum clip(a)clip(b)| <= delta(|clip a|_1 + |clip b|_1) + K delta^2, delta = 1/127."""
    rng = np.random.default_rng(4)
    for K in (8, 64, 512):
        a = rng.normal(0, 1.2, size=(16, K)).astype(np.float32)
        b = rng.normal(0, 0.4, size=(8, K)).astype(np.float32)
        acc = orc.gemm_acc(orc.quantize(a), orc.quantize(b)).astype(np.float64)
        ca, cb = np.clip(a, -2, 2).astype(np.float64), np.clip(b, -2, 2).astype(np.float64)
        exact = ca @ cb.T
        delta = 1.0 / 127.0
        bound = delta * (np.abs(ca).sum(1)[:, None] + np.abs(cb).sum(1)[None, :]) + K * delta * delta
        got = acc * (4.0 / 16129.0)
        assert np.all(np.abs(got - exact) <= bound + 1e-9)


# --------------------------------------------------------------- LN / attention / sigmoid / PE
def test_layernorm_closed_forms(orc):
    d = 64
    g = synth.uniform_activations((d,), 1, 1.0) + np.float32(1)
    b = synth.uniform_activations((d,), 2, 0.5)
    const = np.full(d, 3.25, np.float32)
    assert np.array_equal(orc.layernorm(const, g, b), b)          # LN(const) = beta
    r = synth.uniform_activations((50, d), 3, 4.0)
    out = orc.layernorm(r, np.ones(d, np.float32), np.zeros(d, np.float32)).astype(np.float64)
    v = r.astype(np.float64).var(axis=1)
    assert np.allclose(out.mean(axis=1), 0, atol=1e-6)
    assert np.allclose(out.var(axis=1), v / (v + 1e-6), rtol=1e-5)
    ref = RP.layernorm(r, g, b, 1e-6)
    assert np.mean(orc.layernorm(r, g, b) == ref) > 0.999
    assert np.allclose(orc.layernorm(r, g, b), ref, rtol=1e-6, atol=1e-7)


def test_attention_special_cases(orc):
    d, H = 32, 4
    q = synth.uniform_activations((d,), 5, 1.0)
    K = synth.uniform_activations((7, d), 6, 1.0)
    V = synth.uniform_activations((7, d), 7, 1.0)
    assert np.array_equal(orc.attention(q, K[:1], V[:1], H), V[0])        # S_i = 1 => ctx = v_0
    Keq = np.repeat(K[:1], 7, axis=0)                                       # equal scores => mean
    assert np.allclose(orc.attention(q, Keq, V, H), V.astype(np.float64).mean(0), rtol=1e-6, atol=1e-7)
    ref = RP.attention(q[None], K, V, H)[0]
    assert np.allclose(orc.attention(q, K, V, H), ref, rtol=1e-6, atol=1e-7)
    perm = np.array([3, 0, 6, 1, 5, 2, 4])                                  # permutation invariance
    assert np.allclose(orc.attention(q, K[perm], V[perm], H), orc.attention(q, K, V, H), rtol=1e-6)


def test_sigmoid(orc):
    assert orc.sigmoid(0.0) == 0.5
    for x in (-30.0, -3.5, -0.1, 0.7, 4.0, 20.0):
        assert abs(orc.sigmoid(x) - 1 / (1 + math.exp(-x))) <= 1e-7
        assert abs(orc.sigmoid(-x) - (1 - orc.sigmoid(x))) <= 1e-7


def test_position_encoding(orc):
    d = 16
    p0 = orc.pe(0, d)
    assert np.array_equal(p0, np.tile(np.array([0, 1], np.float32), d // 2))
    p1 = orc.pe(1, d)
    assert p1[0] == np.float32(math.sin(1.0)) and p1[1] == np.float32(math.cos(1.0))
    p = orc.pe(37, 192).astype(np.float64)
    assert np.allclose(p[0::2] ** 2 + p[1::2] ** 2, 1.0, atol=1e-6)
    assert np.array_equal(orc.pe(37, 192), RP.pe_table(38, 192)[37])


# --------------------------------------------------------------- AAN
def test_aan_worked_example(orc):
    G = orc.aan_average(np.array([[2.0], [4.0], [6.0]], np.float32))
    assert G[:, 0].tolist() == [2.0, 3.0, 4.0]
    Y = synth.uniform_activations((1, 8), 2)
    assert np.array_equal(orc.aan_average(Y), Y)                 # T = 1: G = Y


def test_aan_incremental_equals_parallel_and_uniform_attention(orc):
    Y = synth.uniform_activations((40, 24), 12, 3.0)
    G = orc.aan_average(Y)
    t = np.arange(1, 41, dtype=np.float32)[:, None]
    assert np.array_equal(G, np.cumsum(Y, axis=0, dtype=np.float32) / t)   # parallel form
    # masked attention with all-zero scores (uniform weights over 1..t) = average
    zero_q = np.zeros(24, np.float32)
    for tt in (1, 5, 40):
        att = orc.attention(zero_q, Y[:tt], Y[:tt], 1)
        assert np.allclose(G[tt - 1], att, rtol=2e-6, atol=1e-6)
    # exact average in float64: within T*eps of the fp32 running-sum form
    M = np.tril(np.ones((40, 40))) / np.arange(1, 41)[:, None]
    assert np.allclose(G, M @ Y.astype(np.float64), rtol=1e-5, atol=1e-5)


# --------------------------------------------------------------- whole decoder
@pytest.fixture(scope="module")
def tiny_models(orc):
    out = []
    for i, m in enumerate(tiny_variants()):
        w = synth.make_weights(m, seed=100 + i)
        out.append((m, w, orc.OracleModel(m, w), RP.ParallelModel(m, w)))
    return out


def test_encoder_matches_parallel_form(tiny_models):
    for m, w, om, pm in tiny_models:
        src = synth.random_set(1, 9, 9, seed=3, vocab=m.vocab).ids
        e1, kv1 = om.encode(src)
        e2, kv2 = pm.encode(src)
        assert np.allclose(e1, e2, rtol=1e-6, atol=1e-6), m.name
        assert np.allclose(kv1, kv2, rtol=1e-6, atol=1e-6), m.name


def test_teacher_forced_matches_parallel_form(tiny_models):
    """Incremental decoder (carried AAN state / KV cache) == whole-sequence parallel form."""
    for m, w, om, pm in tiny_models:
        for k in range(3):
            ss = synth.random_set(1, 1, 12, seed=20 + k, vocab=m.vocab)
            T = 10
            forced = synth.forced_targets([T], seed=30 + k, vocab=m.vocab)
            ids, tr = om.decode_one(ss.ids, T, forced=forced, trace=True)
            pids, py, _ = pm.forced(ss.ids, forced, T)
            assert np.array_equal(ids, pids), m.name
            assert np.allclose(tr["dec_out"], py, rtol=1e-5, atol=1e-6), m.name
            assert np.mean(tr["dec_out"] == py) > 0.999, m.name


def test_argmax_without_softmax(tiny_models, orc):
    """argmax(logits) == argmax(float64 softmax(logits)) (P:L42 skips softmax)."""
    m, w, om, pm = tiny_models[0]
    ss = synth.random_set(1, 5, 5, seed=8, vocab=m.vocab)
    ids, tr = om.decode_one(ss.ids, 12, forced=synth.forced_targets([12], 9, m.vocab), trace=True)
    qE = orc.quantize(w["emb.E"])
    acc = tr["out_codes"].astype(np.int64) @ qE.astype(np.int64).T
    logits = (acc * np.float64(orc.dequant_scale()) + w["out.b"].astype(np.float64)).astype(np.float32)
    z = logits.astype(np.float64)
    p = np.exp(z - z.max(1, keepdims=True)); p /= p.sum(1, keepdims=True)
    assert np.array_equal(np.argmax(p, axis=1), ids)
    srt = np.sort(logits, axis=1)
    assert np.allclose(tr["margin"], srt[:, -1].astype(np.float64) - srt[:, -2], rtol=0, atol=0)


def test_free_running_equals_full_recompute(tiny_models):
    """Greedy ids with the incremental decoder == re-running the parallel form on the
    whole prefix at every step (brute force, SURVEY 8(c).3 'Incremental decoding')."""
    for m, w, om, pm in tiny_models:
        ss = synth.random_set(1, 3, 10, seed=41, vocab=m.vocab)
        T = 8
        ids = om.decode_one(ss.ids, T)
        prefix = []
        for t in range(1, T + 1):
            pids, _, _ = pm.forced(ss.ids, np.array(prefix, np.int32), t)
            nxt = int(pids[t - 1])
            if nxt == m.eos_id:
                break
            prefix.append(nxt)
        assert ids.tolist() == prefix, m.name


def test_eos_and_max_len(orc):
    m = TINY
    w = synth.make_weights(m, seed=3)
    w["out.b"] = w["out.b"].copy(); w["out.b"][m.eos_id] = 1000.0
    om = orc.OracleModel(m, w)
    src = np.array([5, 6, 7], np.int32)
    assert om.decode_one(src, 10).tolist() == []          # EOS first: nothing emitted
    om2 = orc.OracleModel(m, synth.make_weights(m, seed=3))
    assert om2.decode_one(src, 0).tolist() == []          # max_len 0
    assert len(om2.decode_one(src, 6)) <= 6


def test_vocab_and_state_errors(orc):
    m = TINY
    om = orc.OracleModel(m)
    with pytest.raises(ValueError):
        om.set("enc.0.self.q.W", np.zeros(5, np.float32))     # wrong numel
    with pytest.raises(ValueError):
        om.set("dec.0.self.q.W", np.zeros(32 * 32, np.float32))  # not in an AAN config
    with pytest.raises(ValueError):
        om.quantize()                                      # missing parameters
    om = orc.OracleModel(m, synth.make_weights(m, 1))
    with pytest.raises(ValueError):
        om.decode_one(np.array([64], np.int32), 3)         # id >= V


# --------------------------------------------------------------- Table 1 sizes
@pytest.mark.parametrize("dims,mib", [
    (ModelDims("big", 1024, 4096, 16, decoder=0), 813),
    (ModelDims("base", 512, 2048, 8, decoder=0), 238),
    (ModelDims("small", 256, 2048, 8, decoder=0), 101),
    (ModelDims("tiny192", 192, 1536, 8, aan_ffn_depth=0, aan_gate=0), 60),
    (ModelDims("small-aan", 256, 2048, 8, aan_ffn_depth=1), 100),      # T4 row 15i
    (ModelDims("small-aan-ffn", 256, 2048, 8, aan_ffn_depth=0), 98),   # T3 row 16
    (ModelDims("small-aan-ffn-gate", 256, 2048, 8, aan_ffn_depth=0, aan_gate=0), 95),  # row 17
])
def test_table1_sizes(orc, dims, mib):
    assert orc.param_count(dims) * 4 // 2 ** 20 == mib


# --------------------------------------------------------------- batcher
def test_batcher_at_least_budget(orc):
    order, off = orc.batch_by_words(np.array([5, 3, 2], np.int32), 6)
    assert order.tolist() == [2, 1, 0] and off.tolist() == [0, 3]     # R17: "at least"
    order, off = orc.batch_by_words(np.array([10], np.int32), 6)
    assert order.tolist() == [0] and off.tolist() == [0, 1]
    order, off = orc.batch_by_words(np.zeros(0, np.int32), 6)
    assert off.tolist() == [0]
    with pytest.raises(ValueError):
        orc.batch_by_words(np.array([1], np.int32), 0)


def test_batcher_invariants(orc):
    L = synth.newstest_lengths()
    assert L.sum() == synth.NEWSTEST_TOKENS and len(L) == synth.NEWSTEST_SENTENCES
    for budget in (384, 8192, 65536):
        order, off = orc.batch_by_words(L.astype(np.int32), budget)
        assert sorted(order.tolist()) == list(range(len(L)))           # partition
        Ls = L[order]
        assert np.all(np.diff(Ls) >= 0)                                  # sorted by length
        for b in range(len(off) - 1):
            words = Ls[off[b]:off[b + 1]].sum()
            if b < len(off) - 2:
                assert words >= budget                                   # all but last >= budget
                assert words - Ls[off[b + 1] - 1] < budget               # closed as soon as reached
        # stability: equal lengths keep input order
        for i in range(len(order) - 1):
            if Ls[i] == Ls[i + 1]:
                assert order[i] < order[i + 1]


# --------------------------------------------------------------- exported primitives used by P-1
def test_linear_matches_exact_fma(orc):
    """fmaf((float)acc, s, b): acc*s is exact in float64 (<= 48 significant bits), so one
    float64 add followed by rounding to fp32 equals the fused result (R5)."""
    rng = np.random.default_rng(77)
    qa = rng.integers(-127, 128, size=(9, 96)).astype(np.int8)
    qw = rng.integers(-127, 128, size=(40, 96)).astype(np.int8)
    b = rng.uniform(-0.1, 0.1, 40).astype(np.float32)
    acc = qa.astype(np.int64) @ qw.astype(np.int64).T
    ref = (acc.astype(np.float64) * np.float64(orc.dequant_scale()) + b.astype(np.float64)).astype(np.float32)
    assert np.array_equal(orc.linear(qa, qw, b), ref)
    assert np.array_equal(orc.linear(qa, qw, None),
                          (acc.astype(np.float64) * np.float64(orc.dequant_scale())).astype(np.float32))


def test_residual_ln_gate_form(orc):
    d = 48
    x, dl, gi, gf = (synth.uniform_activations((5, d), s, 2.0) for s in (1, 2, 3, 4))
    gi, gf = orc.sigmoid_array(gi), orc.sigmoid_array(gf)
    g = synth.uniform_activations((d,), 5, 0.1) + np.float32(1)
    b = synth.uniform_activations((d,), 6, 0.1)
    z = gi * x + gf * dl                                  # numpy fp32: one rounding per op
    assert np.allclose(orc.residual_ln(x, dl, g, b, 1e-6, gi, gf), RP.layernorm(x + z, g, b, 1e-6),
                       rtol=1e-6, atol=1e-7)
    assert np.allclose(orc.residual_ln(x, dl, g, b), RP.layernorm(x + dl, g, b, 1e-6), rtol=1e-6, atol=1e-7)


def test_embed_rows(orc):
    E = synth.uniform_activations((20, 16), 8, 0.5)
    out = orc.embed_rows(E, [-1, 3, 19], [0, 5, 7])
    assert np.array_equal(out[0], orc.pe(0, 16))           # start symbol: PE(0) only (R13)
    assert np.array_equal(out[1], RP.embed(E, [3], 5, 16)[0])
    assert np.array_equal(out[2], RP.embed(E, [19], 7, 16)[0])


# --------------------------------------------------------------- bf16 source K/V
def test_bf16_rounding_matches_arithmetic_form(orc):
    """The oracle's bit-pattern rounding == the frexp/rint formulation in tests/ref_parallel.py,
    on random values, exact ties, and values next to ties."""
    rng = np.random.default_rng(5)
    x = np.concatenate([rng.standard_normal(3000).astype(np.float32) * 3,
                        rng.uniform(-1e-30, 1e-30, 200).astype(np.float32),
                        (1 + np.arange(256) / 256.0 + 2.0 ** -9).astype(np.float32),    # ties
                        (1 + np.arange(256) / 256.0 + 2.0 ** -9 + 2.0 ** -22).astype(np.float32)])
    got = np.array([orc.bf16(v) for v in x], np.float32)
    assert np.array_equal(got, RP.bf16_round(x))
    assert np.all(got.view(np.uint32) & 0xFFFF == 0)
    assert np.all(np.abs(got - x) <= np.abs(x) * 2.0 ** -8 + 1e-38)      # half-ulp bound


def test_kv_bf16_oracle_keys_are_bf16_and_rounded_fp32(tiny_models):
    """F3: K/V of a kv_bf16 model are exactly the bf16 rounding of the fp32 model's K/V."""
    for m, w, om, pm in tiny_models:
        if not m.kv_bf16:
            continue
        src = synth.random_set(1, 11, 11, seed=4, vocab=m.vocab).ids
        _, kv16 = om.encode(src)
        m32 = ModelDims(m.name + "-f32", m.d_model, m.d_ffn, m.n_heads, decoder=m.decoder,
                        vocab=m.vocab, enc_layers=m.enc_layers, dec_layers=m.dec_layers)
        _, kv32 = type(om)(m32, w).encode(src)
        assert np.all(kv16.view(np.uint32) & 0xFFFF == 0)
        assert np.array_equal(kv16, RP.bf16_round(kv32))
        assert not np.array_equal(kv16, kv32)
