"""The C-ABI boundary, host logic and isolation rules (no GPU needed)."""
import ast
import os
import re
import subprocess

import numpy as np
import pytest

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libmnmt():
    from paper_1805_12096_b200 import build as B
    B.build()
    from paper_1805_12096_b200 import mnmt as M
    return M


def declared_symbols():
    syms = set()
    for h in ("mnmt.h", "mnmt_ops.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"\b(mnmt_\w+)\s*\(", src):
            syms.add(m.group(1))
    return syms


def test_library_exports_every_declared_symbol(libmnmt):
    out = subprocess.check_output(["nm", "-D", "--defined-only", libmnmt.LIB_PATH], text=True)
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    declared = declared_symbols()
    assert declared, "no declarations parsed"
    assert declared <= exported, declared - exported
    assert declared <= set(libmnmt.EXPORTS)
    L = libmnmt.lib()                                  # loads; resolves every symbol
    for s in declared:
        assert getattr(L, s) is not None


def test_library_is_sm100a_tcgen05(libmnmt):
    sass = subprocess.run(["cuobjdump", "-sass", libmnmt.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", libmnmt.LIB_PATH], capture_output=True,
                                       text=True).stdout or "sm_100a" in sass
    assert "UTCIMMA" in sass          # tcgen05.mma .kind::i8
    assert "UTMALDG" in sass          # TMA loads
    assert "LDTM" in sass             # tcgen05.ld (TMEM -> registers)
    assert "HMMA" not in sass and "IMMA." not in sass.replace("UTCIMMA", "")


def test_host_batcher_matches_oracle(libmnmt, orc):
    L = synth.newstest_lengths()
    for budget in (1, 7, 384, 8192, 65536):
        o1, f1 = libmnmt.batch_by_words(L.astype(np.int32), budget)
        o2, f2 = orc.batch_by_words(L.astype(np.int32), budget)
        assert np.array_equal(o1, o2) and np.array_equal(f1, f2)
    o, f = libmnmt.batch_by_words(np.array([5, 3, 2], np.int32), 6)
    assert o.tolist() == [2, 1, 0] and f.tolist() == [0, 3]
    with pytest.raises(libmnmt.MnmtError) as e:
        libmnmt.batch_by_words(np.array([1], np.int32), 0)
    assert e.value.status == 1


def test_create_without_gpu_fails_loudly(libmnmt):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(libmnmt.MnmtError) as e:
        libmnmt.Model(synth.PRESETS["tiny192-aan"])
    assert e.value.status == 6


def _imports(path):
    tree = ast.parse(open(path).read())
    mods = set()
    for node in ast.walk(tree):
        if isinstance(node, ast.Import):
            mods |= {a.name for a in node.names}
        elif isinstance(node, ast.ImportFrom) and node.module:
            mods.add(node.module)
    return mods


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1805_12096_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            p = os.path.join(dp, f)
            if f.endswith(".py"):
                assert not any(m.startswith("oracle") for m in _imports(p)), p
            if f.endswith((".cu", ".cuh", ".h", ".cpp")):
                assert "oracle" not in open(p).read().lower().replace("oracle's", ""), p


def test_oracle_shares_no_code_with_product():
    src = open(os.path.join(ROOT, "oracle", "mnmt_oracle.c")).read()
    assert "#include \"" not in src                     # only system headers
    for f in ("oracle.py", "__init__.py"):
        assert not any(m.startswith("paper_1805_12096_b200") for m in
                       _imports(os.path.join(ROOT, "oracle", f)))


def test_synth_holds_no_method_arithmetic():
    src = open(os.path.join(ROOT, "synth", "__init__.py")).read()
    for forbidden in ("layernorm", "softmax", "sigmoid", "argmax", "quantiz", "fmaf", "def attn"):
        assert forbidden not in src.lower(), forbidden
