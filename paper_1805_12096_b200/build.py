"""Builds libmnmt.so in-tree with nvcc for sm_100a (no torch involvement)."""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libmnmt.so")
BUILD = os.path.join(HERE, "csrc", "build")
SOURCES = ["gemm_i8.cu", "rowops.cu", "beam.cu", "shortlist.cu", "mnmt.cu", "ops_api.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-fmad=false", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
         "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    srcs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh", ".h"))]
    srcs.append(os.path.join(HERE, "..", "include", "mnmt.h"))
    srcs.append(os.path.join(HERE, "..", "include", "mnmt_ops.h"))
    return any(os.path.getmtime(s) > t for s in srcs)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return OUT
    os.makedirs(BUILD, exist_ok=True)

    def one(src):
        obj = os.path.join(BUILD, src.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        if verbose:
            sys.stderr.write(r.stderr)
        return obj

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(one, SOURCES))
    tmp = OUT + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp,
                           *objs, "-lcudart_static", "-ldl", "-lrt", "-lpthread"])
    os.replace(tmp, OUT)
    return OUT


EXAMPLE_SRC = os.path.join(HERE, "..", "examples", "mnmt_translate.c")
EXAMPLE_BIN = os.path.join(HERE, "..", "examples", "mnmt_translate")


def build_example() -> str:
    """The plain C client of the ABI (examples/mnmt_translate.c), linked against libmnmt.so."""
    if os.path.exists(EXAMPLE_BIN) and os.path.getmtime(EXAMPLE_BIN) >= max(
            os.path.getmtime(EXAMPLE_SRC), os.path.getmtime(OUT)):
        return EXAMPLE_BIN
    subprocess.check_call(["gcc", "-O2", "-Wall", "-std=c11",
                           "-I", os.path.join(HERE, "..", "include"), EXAMPLE_SRC,
                           "-L", HERE, "-lmnmt", "-Wl,-rpath,$ORIGIN/../paper_1805_12096_b200",
                           "-o", EXAMPLE_BIN])
    return EXAMPLE_BIN


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
