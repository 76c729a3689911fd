"""The C ABI from a plain C program (examples/mnmt_translate.c, no Python in the process):
it builds and links against libmnmt.so here; on a B200 its ids equal the oracle's
(greedy and with a batch shortlist)."""
import os
import subprocess

import numpy as np
import pytest

import synth
from synth import ModelDims

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def client():
    from paper_1805_12096_b200 import build as B
    B.build()
    return B.build_example()


def test_builds_links_and_reports_usage():
    r = subprocess.run([client()], capture_output=True, text=True)
    assert r.returncode == 1 and "usage" in r.stderr


def _gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.gpu
@pytest.mark.skipif(not _gpu(), reason="needs a B200")
@pytest.mark.parametrize("dims", [
    ModelDims("t-aan", 32, 64, 4, vocab=64, enc_layers=2, dec_layers=2),
    ModelDims("t192-self", 192, 384, 8, vocab=1000, enc_layers=2, dec_layers=2, decoder=0),
], ids=lambda d: d.name)
@pytest.mark.parametrize("shortlist", [False, True])
def test_c_client_matches_oracle(tmp_path, dims, shortlist):
    import oracle.oracle as O
    w = synth.make_weights(dims, seed=51, emb_scale=0.05)
    ss = synth.random_set(23, 1, 15, seed=17, vocab=dims.vocab)
    synth.write_weights_bin(str(tmp_path / "w.bin"), dims, w)
    synth.write_sentences_bin(str(tmp_path / "s.bin"), ss)
    budget = 40
    args = [client(), str(tmp_path / "w.bin"), str(tmp_path / "s.bin"), str(dims.d_model),
            str(dims.d_ffn), str(dims.n_heads), str(dims.enc_layers), str(dims.vocab),
            str(dims.decoder), str(dims.aan_ffn_depth), str(dims.aan_gate), str(budget)]
    om = O.OracleModel(dims, w)
    if shortlist:
        freq, lex = synth.shortlist_tables(dims.vocab, 8, 4, seed=3)
        synth.write_shortlist_bin(str(tmp_path / "l.bin"), freq, lex)
        args.append(str(tmp_path / "l.bin"))
        order, off = O.batch_by_words(ss.lengths, budget)
        ref = [None] * ss.n
        for b in range(len(off) - 1):
            idx = order[off[b]:off[b + 1]]
            sub = ss.subset(idx)
            sl = O.build_shortlist(dims.vocab, freq, lex, sub.ids)
            for i, ids in zip(idx, om.decode_many_sl(sub, sl, 4)):
                ref[i] = ids
    else:
        ref = om.decode_many(ss, 4)
    r = subprocess.run(args, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.split("\n")[:ss.n]
    got = [np.array([int(t) for t in ln.split()], np.int32) for ln in lines]
    assert all(np.array_equal(a, b) for a, b in zip(got, ref))
