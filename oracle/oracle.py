"""ctypes wrapper of liboracle.so (TEST INFRASTRUCTURE ONLY — see __init__.py).

Argument marshalling only; every computation is in mnmt_oracle.c.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Dict, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mnmt_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile the oracle (plain gcc; no CUDA)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class Cfg(C.Structure):
    _fields_ = [("d_model", C.c_int32), ("d_ffn", C.c_int32), ("n_heads", C.c_int32),
                ("enc_layers", C.c_int32), ("dec_layers", C.c_int32), ("vocab", C.c_int32),
                ("decoder", C.c_int32), ("aan_ffn_depth", C.c_int32), ("aan_gate", C.c_int32),
                ("out_bias", C.c_int32), ("eos_id", C.c_int32), ("clip", C.c_float),
                ("ln_eps", C.c_float), ("arith", C.c_int32), ("src_kv_bf16", C.c_int32)]


class Trace(C.Structure):
    _fields_ = [("ids", C.c_void_p), ("second", C.c_void_p), ("margin", C.c_void_p),
                ("dec_out", C.c_void_p), ("layer_out", C.c_void_p), ("out_codes", C.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        P = C.c_void_p
        L.orc_sigma.restype = C.c_float; L.orc_sigma.argtypes = [C.c_float]
        L.orc_dequant_scale.restype = C.c_float; L.orc_dequant_scale.argtypes = [C.c_float]
        L.orc_q.restype = C.c_int8; L.orc_q.argtypes = [C.c_float, C.c_float]
        L.orc_quantize.argtypes = [P, C.c_int64, C.c_float, P]
        L.orc_gemm_acc.argtypes = [P, P, C.c_int, C.c_int, C.c_int, P]
        L.orc_layernorm.argtypes = [P, C.c_int, P, P, C.c_float, P]
        L.orc_attention.argtypes = [P, P, P, C.c_int64, C.c_int, C.c_int, C.c_int, P]
        L.orc_sigmoid.restype = C.c_float; L.orc_sigmoid.argtypes = [C.c_float]
        L.orc_pe.argtypes = [C.c_int, C.c_int, P]
        L.orc_aan_step.argtypes = [P, P, C.c_int, C.c_int, P]
        L.orc_linear.argtypes = [P, P, C.c_int, C.c_int, C.c_int, P, C.c_float, P]
        L.orc_sigmoid_array.argtypes = [P, C.c_int64, P]
        L.orc_residual_ln.argtypes = [P, P, P, P, C.c_int, P, P, C.c_float, P]
        L.orc_embed_row.argtypes = [P, C.c_int, C.c_int, C.c_int, P]
        L.orc_model_new.restype = P; L.orc_model_new.argtypes = [C.POINTER(Cfg)]
        L.orc_model_free.argtypes = [P]
        L.orc_model_set.restype = C.c_int; L.orc_model_set.argtypes = [P, C.c_char_p, P, C.c_int64]
        L.orc_model_quantize.restype = C.c_int; L.orc_model_quantize.argtypes = [P]
        L.orc_encode.restype = C.c_int; L.orc_encode.argtypes = [P, P, C.c_int, P, P]
        L.orc_decode_one.restype = C.c_int
        L.orc_decode_one.argtypes = [P, P, C.c_int, C.c_int, P, P, C.POINTER(Trace)]
        L.orc_decode_many.restype = C.c_int
        L.orc_decode_many.argtypes = [P, P, P, C.c_int, P, P, P, C.c_int]
        L.orc_beam_one.restype = C.c_int
        L.orc_beam_one.argtypes = [P, P, C.c_int, C.c_int, C.c_int, P, P, P]
        L.orc_beam_many.restype = C.c_int
        L.orc_beam_many.argtypes = [P, P, P, C.c_int, P, C.c_int, P, P, P, P, C.c_int]
        L.orc_bf16.restype = C.c_float
        L.orc_bf16.argtypes = [C.c_float]
        L.orc_build_shortlist.restype = C.c_int
        L.orc_build_shortlist.argtypes = [C.c_int, P, C.c_int, P, C.c_int, P, C.c_int64, C.c_int,
                                          C.c_int, P]
        L.orc_decode_many_sl.restype = C.c_int
        L.orc_decode_many_sl.argtypes = [P, P, P, C.c_int, P, P, C.c_int, P, P, C.c_int]
        L.orc_q16.restype = C.c_int16; L.orc_q16.argtypes = [C.c_float]
        L.orc_dot_codes.restype = C.c_int32; L.orc_dot_codes.argtypes = [C.c_int, P, P, C.c_int]
        L.orc_logsumexp.restype = C.c_float
        L.orc_logsumexp.argtypes = [P, C.c_int]
        L.orc_max_threads.restype = C.c_int
        L.orc_batch_by_words.restype = C.c_int
        L.orc_batch_by_words.argtypes = [P, C.c_int, C.c_int, P, P, P]
        L.orc_param_count.restype = C.c_int64; L.orc_param_count.argtypes = [C.POINTER(Cfg)]
    return _lib


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# Integer arithmetic of the products (oracle only): the GPU path is ARITH_S32.
ARITH_S32, ARITH_SAT16, ARITH_INT16 = 0, 1, 2


def cfg_from_dims(m, arith: int = ARITH_S32) -> Cfg:
    return Cfg(m.d_model, m.d_ffn, m.n_heads, m.enc_layers, m.dec_layers, m.vocab, m.decoder,
               m.aan_ffn_depth, m.aan_gate, m.out_bias, m.eos_id, m.clip, m.ln_eps, arith,
               getattr(m, "kv_bf16", 0))


def q16(x: float) -> int:
    """int16 code RNE(x * 2^10), saturated."""
    return int(lib().orc_q16(float(x)))


def dot_codes(arith: int, a, w) -> int:
    """One dot product of codes under the given arithmetic (0 exact, 1 sat16 pairs, 2 wrap32)."""
    a = np.ascontiguousarray(a, dtype=np.int16); w = np.ascontiguousarray(w, dtype=np.int16)
    assert a.shape == w.shape
    return int(lib().orc_dot_codes(int(arith), _p(a), _p(w), a.size))


# ------------------------------------------------------------------ scalars / kernels
def bf16(x: float) -> float:
    """Nearest bfloat16 of a finite fp32 value, ties to even (F3, R35)."""
    return float(lib().orc_bf16(float(np.float32(x))))


def sigma(clip: float = 2.0) -> float:
    return lib().orc_sigma(clip)


def dequant_scale(clip: float = 2.0) -> float:
    return lib().orc_dequant_scale(clip)


def quantize(x: np.ndarray, clip: float = 2.0) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty(x.shape, dtype=np.int8)
    lib().orc_quantize(_p(x), x.size, clip, _p(out))
    return out


def gemm_acc(a: np.ndarray, w: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.int8); w = np.ascontiguousarray(w, dtype=np.int8)
    M, K = a.shape; N, K2 = w.shape
    assert K == K2
    out = np.empty((M, N), dtype=np.int32)
    lib().orc_gemm_acc(_p(a), _p(w), M, N, K, _p(out))
    return out


def linear(qa: np.ndarray, qw: np.ndarray, bias: Optional[np.ndarray], clip: float = 2.0) -> np.ndarray:
    """lin(qa; W, b) = fmaf((float)acc, s, b) over rows of qa [M x K], qw [N x K]."""
    qa = np.ascontiguousarray(qa, dtype=np.int8); qw = np.ascontiguousarray(qw, dtype=np.int8)
    M, K = qa.shape; N = qw.shape[0]
    b = None if bias is None else np.ascontiguousarray(bias, dtype=np.float32)
    out = np.empty((M, N), np.float32)
    lib().orc_linear(_p(qa), _p(qw), M, N, K, _p(b), clip, _p(out))
    return out


def sigmoid_array(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty_like(x)
    lib().orc_sigmoid_array(_p(x), x.size, _p(out))
    return out


def residual_ln(x, delta, g, b, eps=1e-6, gi=None, gf=None) -> np.ndarray:
    """Rows: LN(fl(x + delta)) or the gate form LN(fl(x + fl(fl(gi*x) + fl(gf*delta))))."""
    x = np.ascontiguousarray(x, np.float32); delta = np.ascontiguousarray(delta, np.float32)
    g = np.ascontiguousarray(g, np.float32); b = np.ascontiguousarray(b, np.float32)
    if gi is not None:
        gi = np.ascontiguousarray(gi, np.float32); gf = np.ascontiguousarray(gf, np.float32)
    d = x.shape[-1]
    out = np.empty_like(x)
    for i in range(x.shape[0]):
        lib().orc_residual_ln(_p(x[i]), _p(delta[i]), _p(None if gi is None else gi[i]),
                              _p(None if gf is None else gf[i]), d, _p(g), _p(b), eps, _p(out[i]))
    return out


def embed_rows(E: np.ndarray, ids, pos) -> np.ndarray:
    E = np.ascontiguousarray(E, np.float32)
    d = E.shape[1]
    out = np.empty((len(ids), d), np.float32)
    for i, (t, p) in enumerate(zip(ids, pos)):
        lib().orc_embed_row(_p(E), d, int(t), int(p), _p(out[i]))
    return out


def layernorm(r: np.ndarray, g: np.ndarray, b: np.ndarray, eps: float = 1e-6) -> np.ndarray:
    r = np.ascontiguousarray(r, dtype=np.float32)
    g = np.ascontiguousarray(g, dtype=np.float32); b = np.ascontiguousarray(b, dtype=np.float32)
    out = np.empty_like(r)
    d = r.shape[-1]
    rr = r.reshape(-1, d); oo = out.reshape(-1, d)
    for i in range(rr.shape[0]):
        lib().orc_layernorm(_p(rr[i]), d, _p(g), _p(b), eps, _p(oo[i]))
    return out


def attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, H: int) -> np.ndarray:
    """One query row q [d] over key/value rows k, v [n x d]."""
    q = np.ascontiguousarray(q, dtype=np.float32)
    k = np.ascontiguousarray(k, dtype=np.float32); v = np.ascontiguousarray(v, dtype=np.float32)
    d = q.shape[0]; n = k.shape[0]
    ctx = np.empty(d, dtype=np.float32)
    lib().orc_attention(_p(q), _p(k), _p(v), d, n, d, H, _p(ctx))
    return ctx


def sigmoid(x: float) -> float:
    return lib().orc_sigmoid(float(x))


def pe(pos: int, d: int) -> np.ndarray:
    out = np.empty(d, dtype=np.float32)
    lib().orc_pe(pos, d, _p(out))
    return out


def aan_average(Y: np.ndarray) -> np.ndarray:
    """Run the incremental AAN recurrence over rows of Y [T x d]; returns G [T x d]."""
    Y = np.ascontiguousarray(Y, dtype=np.float32)
    T, d = Y.shape
    Cst = np.zeros(d, np.float32); G = np.empty_like(Y)
    for t in range(T):
        lib().orc_aan_step(_p(Cst), _p(Y[t]), t + 1, d, _p(G[t]))
    return G


def batch_by_words(lengths: np.ndarray, budget: int):
    lengths = np.ascontiguousarray(lengths, dtype=np.int32)
    n = lengths.shape[0]
    order = np.empty(max(n, 1), dtype=np.int32); off = np.empty(n + 2, dtype=np.int32)
    nb = np.zeros(1, dtype=np.int32)
    st = lib().orc_batch_by_words(_p(lengths), n, budget, _p(order), _p(off), _p(nb))
    if st:
        raise ValueError("batch_by_words: bad argument")
    return order[:n].copy(), off[:nb[0] + 1].copy()


def param_count(m) -> int:
    c = cfg_from_dims(m)
    return int(lib().orc_param_count(C.byref(c)))


# ------------------------------------------------------------------ model
class OracleModel:
    """The oracle's model: set every parameter, quantize once."""

    def __init__(self, dims, weights: Optional[Dict[str, np.ndarray]] = None, arith: int = ARITH_S32):
        self.dims = dims
        self._cfg = cfg_from_dims(dims, arith)
        self.h = lib().orc_model_new(C.byref(self._cfg))
        if not self.h:
            raise ValueError("oracle: bad config")
        if weights is not None:
            for k, v in weights.items():
                self.set(k, v)
            self.quantize()

    def set(self, name: str, arr: np.ndarray) -> None:
        a = np.ascontiguousarray(arr, dtype=np.float32)
        st = lib().orc_model_set(self.h, name.encode(), _p(a), a.size)
        if st:
            raise ValueError(f"oracle: set {name}: status {st}")

    def quantize(self) -> None:
        st = lib().orc_model_quantize(self.h)
        if st:
            raise ValueError(f"oracle: quantize status {st}")

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().orc_model_free(self.h)
                self.h = None
        except Exception:
            pass

    def encode(self, src: np.ndarray):
        """Returns (enc_out [S x d], kv [L][2][S][d])."""
        src = np.ascontiguousarray(src, dtype=np.int32)
        S = src.shape[0]; d = self.dims.d_model; L = self.dims.dec_layers
        enc = np.empty((S, d), np.float32); kv = np.empty((L, 2, S, d), np.float32)
        st = lib().orc_encode(self.h, _p(src), S, _p(enc), _p(kv))
        if st:
            raise ValueError(f"oracle: encode status {st}")
        return enc, kv

    def decode_one(self, src: np.ndarray, max_len: int, forced: Optional[np.ndarray] = None,
                   trace: bool = False, layers: bool = False):
        src = np.ascontiguousarray(src, dtype=np.int32)
        d = self.dims.d_model; L = self.dims.dec_layers
        T = max(max_len, 0)
        out = np.zeros(max(T, 1), np.int32)
        tr = None; res = {}
        if trace:
            res = dict(ids=np.zeros(T, np.int32), second=np.zeros(T, np.int32),
                       margin=np.zeros(T, np.float32), dec_out=np.zeros((T, d), np.float32),
                       out_codes=np.zeros((T, d), np.int8))
            if layers:
                res["layer_out"] = np.zeros((T, L, 3, d), np.float32)
            tr = Trace(_p(res["ids"]), _p(res["second"]), _p(res["margin"]), _p(res["dec_out"]),
                       _p(res.get("layer_out")), _p(res["out_codes"]))
        f = None
        if forced is not None:
            f = np.ascontiguousarray(forced, dtype=np.int32)
            if f.size == 0:
                f = np.zeros(1, np.int32)
        n = lib().orc_decode_one(self.h, _p(src), src.shape[0], T, _p(f), _p(out),
                                 C.byref(tr) if tr is not None else None)
        if n < 0:
            raise ValueError(f"oracle: decode status {-n}")
        ids = out[:n].copy()
        return (ids, res) if trace else ids

    def beam_one(self, src: np.ndarray, max_len: int, beam: int):
        """Beam search of one sentence (R26-R29).
        Returns [(ids, score)] sorted by descending score (<= beam entries)."""
        src = np.ascontiguousarray(src, dtype=np.int32)
        T = max(int(max_len), 0)
        ids = np.zeros(max(beam * T, 1), np.int32)
        ln = np.zeros(beam, np.int32)
        sc = np.zeros(beam, np.float32)
        n = lib().orc_beam_one(self.h, _p(src), src.shape[0], T, int(beam), _p(ids), _p(ln), _p(sc))
        if n < 0:
            raise ValueError(f"oracle: beam status {-n}")
        return [(ids[r * T:r * T + ln[r]].copy(), float(sc[r])) for r in range(n)]

    def beam_many(self, sset, beam: int, nthreads: int = 0):
        """Beam search of every sentence of a SentenceSet; list of n-best lists."""
        n = sset.n
        ml = np.ascontiguousarray(sset.max_len, dtype=np.int32)
        ids = np.zeros(max(int(ml.sum()) * beam, 1), np.int32)
        ln = np.zeros(max(n * beam, 1), np.int32)
        sc = np.zeros(max(n * beam, 1), np.float32)
        nh = np.zeros(max(n, 1), np.int32)
        src = np.ascontiguousarray(sset.ids, dtype=np.int32)
        offs = np.ascontiguousarray(sset.offsets, dtype=np.int64)
        st = lib().orc_beam_many(self.h, _p(src), _p(offs), n, _p(ml), int(beam), _p(ids), _p(ln),
                                 _p(sc), _p(nh), nthreads)
        if st:
            raise ValueError(f"oracle: beam_many status {st}")
        res = []
        o = 0
        for i in range(n):
            T = int(ml[i])
            res.append([(ids[beam * o + r * T: beam * o + r * T + ln[i * beam + r]].copy(),
                         float(sc[i * beam + r])) for r in range(nh[i])])
            o += T
        return res

    def decode_many_sl(self, sset, shortlist: np.ndarray, nthreads: int = 0):
        """decode_many with every sentence restricted to `shortlist` (one batch, F2)."""
        n = sset.n
        ml = np.ascontiguousarray(sset.max_len, dtype=np.int32)
        out = np.zeros(max(int(ml.sum()), 1), np.int32)
        out_len = np.zeros(max(n, 1), np.int32)
        ids = np.ascontiguousarray(sset.ids, dtype=np.int32)
        offs = np.ascontiguousarray(sset.offsets, dtype=np.int64)
        sl = np.ascontiguousarray(shortlist, dtype=np.int32)
        st = lib().orc_decode_many_sl(self.h, _p(ids), _p(offs), n, _p(ml), _p(sl), sl.size,
                                      _p(out), _p(out_len), nthreads)
        if st:
            raise ValueError(f"oracle: decode_many_sl status {st}")
        res, o = [], 0
        for i in range(n):
            res.append(out[o:o + out_len[i]].copy())
            o += int(ml[i])
        return res

    def decode_many(self, sset, nthreads: int = 0):
        """Free-running greedy decode of a SentenceSet; returns list of id arrays."""
        n = sset.n
        ml = np.ascontiguousarray(sset.max_len, dtype=np.int32)
        out = np.zeros(max(int(ml.sum()), 1), np.int32)
        out_len = np.zeros(max(n, 1), np.int32)
        ids = np.ascontiguousarray(sset.ids, dtype=np.int32)
        offs = np.ascontiguousarray(sset.offsets, dtype=np.int64)
        st = lib().orc_decode_many(self.h, _p(ids), _p(offs), n, _p(ml), _p(out), _p(out_len),
                                   nthreads)
        if st:
            raise ValueError(f"oracle: decode_many status {st}")
        res = []
        o = 0
        for i in range(n):
            res.append(out[o:o + out_len[i]].copy())
            o += int(ml[i])
        return res


def build_shortlist(V: int, freq: np.ndarray, lex: np.ndarray, src_ids: np.ndarray,
                    eos: int = 0, unk: int = 1) -> np.ndarray:
    """Batch shortlist: freq ∪ lex rows of the batch's source ids ∪ {EOS,
    UNK}, ascending.  lex: [V x k_lex] int32."""
    freq = np.ascontiguousarray(freq, np.int32)
    lex = np.ascontiguousarray(lex, np.int32)
    src = np.ascontiguousarray(src_ids, np.int32)
    out = np.zeros(V, np.int32)
    n = lib().orc_build_shortlist(V, _p(freq), freq.size, _p(lex), lex.shape[1] if lex.ndim == 2 else 0,
                                  _p(src), src.size, eos, unk, _p(out))
    return out[:n].copy()


def logsumexp(logits: np.ndarray) -> float:
    """fl32(M + log sum_j exp(l_j - M)) of one row (reading R26)."""
    l = np.ascontiguousarray(logits, dtype=np.float32)
    return float(lib().orc_logsumexp(_p(l), l.size))


def max_threads() -> int:
    return int(lib().orc_max_threads())
