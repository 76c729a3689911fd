"""P-0 pins of the CPU oracle against the values PAPER.md / SPEC.md print, read from the cited
text fixtures under tests/golden/ (one fixture line per printed value)."""
import os

import numpy as np
import pytest

from synth import ModelDims

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def rows(name):
    """Non-comment lines of a fixture, whitespace-split."""
    with open(os.path.join(GOLDEN, name)) as f:
        return [ln.split() for ln in f if ln.strip() and not ln.lstrip().startswith("#")]


def test_fixtures_cite_their_passage():
    for name in os.listdir(GOLDEN):
        if name.endswith(".txt"):
            for r in rows(name):
                assert any("PAPER.md:L" in t or "SPEC.md:L" in t for t in r), (name, r)


@pytest.mark.parametrize("r", rows("table1_sizes.txt"), ids=lambda r: r[0])
def test_table1_sizes(orc, r):
    name, d, F, H, dec, depth, gate, mib = r[0], *map(int, r[1:8])
    dims = ModelDims(name, d, F, H, decoder=dec, aan_ffn_depth=depth, aan_gate=gate)
    assert orc.param_count(dims) * 4 // 2 ** 20 == mib


def test_quantizer_examples(orc):
    rs = rows("quantizer_examples.txt")
    x = np.array([float(r[0]) for r in rs], np.float32)
    assert orc.quantize(x).tolist() == [int(r[1]) for r in rs]


def test_gemm_i8_example(orc):
    for r in rows("gemm_i8_example.txt"):
        a, b, acc, res, tol = float(r[0]), float(r[1]), int(r[2]), float(r[3]), float(r[4])
        qa = orc.quantize(np.array([[a, 0.0]], np.float32))     # k padded to 2 with a zero
        qb = orc.quantize(np.array([[b, 0.0]], np.float32))
        got = orc.gemm_acc(qa, qb)[0, 0]
        assert got == acc
        assert abs(float(got) * orc.dequant_scale() - res) < tol


def test_aan_average_example(orc):
    rs = rows("aan_average_example.txt")
    Y = np.array([[float(r[0])] for r in rs], np.float32)
    assert orc.aan_average(Y)[:, 0].tolist() == [float(r[1]) for r in rs]


def _ids(spec, V):
    if not spec:
        return []
    out = []
    for part in spec.split(","):
        if ".." in part:
            a, b = map(int, part.split(".."))
            out += list(range(a, b + 1)) if a <= b else list(range(a, b - 1, -1))
        else:
            out.append(int(part))
    return out


def test_shortlist_examples(orc):
    with open(os.path.join(GOLDEN, "shortlist_examples.txt")) as f:
        cases = [ln for ln in f if ln.startswith("case ")]
    assert cases
    for ln in cases:
        fields = {}
        for p in ln.split("|")[1:]:
            if "=" in p:
                k, v = p.strip().split("=", 1)
                fields[k] = v.strip()
        V = int(fields["V"])
        lex_rows = {}
        for item in filter(None, fields["lex"].split(";")):
            s, ts = item.split(":")
            lex_rows[int(s)] = [int(t) for t in ts.split(",")]
        k = max((len(v) for v in lex_rows.values()), default=3)
        lex = np.full((V, k), V - 1, np.int32)
        for s, ts in lex_rows.items():
            lex[s] = ts
        freq = np.array(_ids(fields["freq"], V), np.int32)
        src = np.array(_ids(fields["src"], V), np.int32)
        got = orc.build_shortlist(V, freq, lex, src)
        assert got.tolist() == _ids(fields["expect"], V), ln


def test_bf16_rounding_examples(orc):
    for r in rows("bf16_rounding.txt"):
        assert orc.bf16(float(r[0])) == float(r[1]), r
