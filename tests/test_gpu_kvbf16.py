"""bf16 source keys / values (R35): libmnmt with
src_kv_bf16 = 1 against the oracle with the same flag (tests/test_oracle_pins.py pins the
oracle's rounding and its bf16 decoder against an independent formulation).

Bar: as the fp32 path (tests/test_gpu_model.py): teacher-forced per-step ids bit-exact, encoder
output / source K,V (now bf16 values) / every decoder layer within tolerance, free-running ids
identical, on every engine and through the split source-attention kernels.
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
from tests.test_gpu_model import forced_case, run_forced_parity  # noqa: E402

VARIANTS = [
    ModelDims("t-aan-kv16", 32, 64, 4, vocab=64, enc_layers=2, dec_layers=2, kv_bf16=1),
    ModelDims("t-self-kv16", 32, 64, 4, vocab=64, enc_layers=2, dec_layers=2, decoder=0, kv_bf16=1),
    ModelDims("t-nobias-kv16", 48, 96, 4, vocab=50, enc_layers=1, dec_layers=3, out_bias=0,
              kv_bf16=1),
    ModelDims("t192-aan-kv16", 192, 384, 8, vocab=1000, enc_layers=2, dec_layers=2, kv_bf16=1),
    ModelDims("t256-self-kv16", 256, 512, 8, vocab=1000, enc_layers=2, dec_layers=2, decoder=0,
              kv_bf16=1),
]


def pair(dims, seed):
    w = synth.make_weights(dims, seed=seed)
    return w, O.OracleModel(dims, w), M.Model(dims, w)


@pytest.mark.parametrize("dims", VARIANTS, ids=lambda d: d.name)
def test_teacher_forced(dims):
    w, om, gm = pair(dims, 11)
    ss, forced, foff = forced_case(dims, 9, 0, 13, 0, 17, seed=3)
    tot, ex, fl = run_forced_parity(dims, w, om, gm, ss, forced, foff)
    assert ex == tot, f"{tot - ex} flagged near-ties"
    _, dumps = gm.decode_forced(ss, forced, foff, M.DUMP_SRC_KV)
    assert np.all(dumps["src_kv"].view(np.uint32) & 0xFFFF == 0)      # bf16 values


@pytest.mark.parametrize("lo,hi", [(30, 90), (60, 140)], ids=["split2", "split4"])
def test_long_sources_split_attention(lo, hi):
    dims = VARIANTS[0]
    w, om, gm = pair(dims, 21)
    ss, forced, foff = forced_case(dims, 7, lo, hi, 2, 6, seed=9)
    tot, ex, fl = run_forced_parity(dims, w, om, gm, ss, forced, foff)
    assert ex == tot, f"{tot - ex} flagged near-ties"


@pytest.mark.parametrize("dims", VARIANTS, ids=lambda d: d.name)
def test_free_running(dims):
    w, om, gm = pair(dims, 12)
    ss = synth.random_set(17, 1, 70, seed=5, vocab=dims.vocab)
    ref = om.decode_many(ss, 4)
    got = gm.decode(ss)
    assert all(np.array_equal(a, b) for a, b in zip(got, ref))


def test_differs_from_fp32_and_bench_options():
    """The flag changes the model (ids differ from the fp32 K/V model somewhere), and the bench
    launch options change no id."""
    dims = ModelDims("t192-aan-kv16", 192, 384, 8, vocab=1000, enc_layers=2, dec_layers=2,
                     kv_bf16=1)
    w = synth.make_weights(dims, seed=14, emb_scale=0.05)
    om, gm = O.OracleModel(dims, w), M.Model(dims, w)
    ss = synth.random_set(80, 1, 60, seed=6, vocab=dims.vocab)
    ref = om.decode_many(ss, 4)
    for name, v in [("lanes", 3), ("lane_tiers", 40), ("max_concurrent_rows", 4096),
                    ("green_sms", 48), ("pers_reserve", 16)]:
        gm.set_option(name, v)
    got = gm.translate(ss, 200)
    assert all(np.array_equal(a, b) for a, b in zip(got, ref))
    d32 = ModelDims("t192-aan", 192, 384, 8, vocab=1000, enc_layers=2, dec_layers=2)
    ref32 = O.OracleModel(d32, w).decode_many(ss, 4)
    assert any(not np.array_equal(a, b) for a, b in zip(ref, ref32))


def test_small_aan_newstest_sampled():
    """configs[1] model with bf16 K/V: a sample of the newstest-shaped set, ids identical."""
    dims = synth.PRESETS["small-aan"]
    dims = ModelDims("small-aan-kv16", dims.d_model, dims.d_ffn, dims.n_heads, kv_bf16=1)
    w = synth.make_weights(dims, seed=1)
    om, gm = O.OracleModel(dims, w), M.Model(dims, w)
    ss = synth.newstest_set().subset(np.arange(0, 3003, 100))
    got = gm.translate(ss, 8192)
    ref = om.decode_many(ss, 0)
    assert all(np.array_equal(a, b) for a, b in zip(got, ref))
