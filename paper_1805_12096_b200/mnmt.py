"""ctypes binding of libmnmt (include/mnmt.h, include/mnmt_ops.h).

Argument marshalling only: every step of the decode path runs in the sm_100a
kernels of libmnmt.so.  There is no fallback: if the in-tree library is
missing or fails to load, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmnmt.so")

ABI_VERSION = 2
MAX_SPAN = 512
DEVICE_IO = 1
SHORTLIST = 2

DUMP_ENC_OUT, DUMP_SRC_KV, DUMP_DEC_OUT, DUMP_OUT_CODES, DUMP_LAYERS, DUMP_MARGIN = 1, 2, 4, 8, 16, 32
EPI_F32, EPI_F32_Q, EPI_RELU_Q, EPI_RELU_F32_Q, EPI_SIGMOID, EPI_ARGMAX, EPI_ACC = range(7)
EPI_TOPK = 9            # beam search partials (include/mnmt_ops.h); 80-byte records
TOPK_RECORD_BYTES = 80

STATUS = {0: "OK", 1: "ERR_ARG", 2: "ERR_DIM", 3: "ERR_VOCAB", 4: "ERR_STATE",
          5: "ERR_CAPACITY", 6: "ERR_CUDA", 7: "ERR_OOM"}


class MnmtError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Config(C.Structure):
    _fields_ = [("abi_version", C.c_int32), ("d_model", C.c_int32), ("d_ffn", C.c_int32),
                ("n_heads", C.c_int32), ("enc_layers", C.c_int32), ("dec_layers", C.c_int32),
                ("vocab", C.c_int32), ("decoder", C.c_int32), ("aan_ffn_depth", C.c_int32),
                ("aan_gate", C.c_int32), ("out_bias", C.c_int32), ("eos_id", C.c_int32),
                ("clip", C.c_float), ("ln_eps", C.c_float), ("src_kv_bf16", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("gpu_launches", C.c_int64), ("decode_steps", C.c_int64), ("batches", C.c_int64),
                ("target_words", C.c_int64), ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64)]


EXPORTS = [
    "mnmt_config_default", "mnmt_model_create", "mnmt_model_set_param", "mnmt_model_quantize",
    "mnmt_batch_by_words", "mnmt_decode", "mnmt_translate", "mnmt_beam_translate",
    "mnmt_model_set_shortlist",
    "mnmt_decode_forced", "mnmt_translate_forced",
    "mnmt_get_stats", "mnmt_last_error", "mnmt_model_destroy", "mnmt_model_set_option",
    "mnmt_op_quantize", "mnmt_op_gemm_i8", "mnmt_op_argmax_ids", "mnmt_op_layernorm",
    "mnmt_op_aan_step", "mnmt_op_embed", "mnmt_op_attention", "mnmt_op_attention_enc", "mnmt_op_attention_bf16",
    "mnmt_op_gather_rows", "mnmt_op_src_attention", "mnmt_op_src_attention_f32", "mnmt_op_gemm_i8_split",
]

_lib = None


def lib():
    """Loads the in-tree libmnmt.so (raises if it is missing: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libmnmt.so not built ({LIB_PATH}); run __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    P, I32, I64, F = C.c_void_p, C.c_int32, C.c_int64, C.c_float
    S = C.c_int
    L.mnmt_config_default.argtypes = [C.POINTER(Config), I32, I32, I32]
    L.mnmt_config_default.restype = None
    L.mnmt_model_create.argtypes = [C.POINTER(Config), I32, C.POINTER(P)]
    L.mnmt_model_set_param.argtypes = [P, C.c_char_p, P, I64]
    L.mnmt_model_quantize.argtypes = [P]
    L.mnmt_batch_by_words.argtypes = [P, I32, I32, P, P, P]
    L.mnmt_decode.argtypes = [P, P, P, I32, P, P, I64, P, P]
    L.mnmt_translate.argtypes = [P, P, P, I32, P, I32, P, I64, P, C.c_uint32, P]
    L.mnmt_model_set_shortlist.argtypes = [P, P, I32, P, I32]
    L.mnmt_beam_translate.argtypes = [P, P, P, I32, P, I32, I32, P, I64, P, P, P, C.c_uint32, P]
    L.mnmt_decode_forced.argtypes = [P, P, P, I32, P, P, P, C.c_uint32, P, I64, P]
    L.mnmt_translate_forced.argtypes = [P, P, P, I32, P, P, I32, P, C.c_uint32, P, I64, P]
    L.mnmt_get_stats.argtypes = [P, C.POINTER(Stats)]
    L.mnmt_model_set_option.argtypes = [P, C.c_char_p, I64]
    L.mnmt_last_error.argtypes = []
    L.mnmt_last_error.restype = C.c_char_p
    L.mnmt_model_destroy.argtypes = [P]
    L.mnmt_model_destroy.restype = None
    L.mnmt_op_quantize.argtypes = [P, I64, F, P, P]
    L.mnmt_op_gemm_i8.argtypes = [P, P, I32, I32, I32, P, F, I32, P, P, I32, P]
    L.mnmt_op_argmax_ids.argtypes = [P, I32, P, P]
    L.mnmt_op_layernorm.argtypes = [P, P, P, P, P, P, I32, I32, F, F, P, P, P]
    L.mnmt_op_aan_step.argtypes = [P, P, I32, I32, I32, F, P, P, P]
    L.mnmt_op_embed.argtypes = [P, I32, P, P, I32, F, P, P, P]
    L.mnmt_op_attention.argtypes = [P, I64, P, I64, I32, I32, P, P, I32, I32, I32, F, P, P, P]
    L.mnmt_op_attention_enc.argtypes = [P, P, P, I32, I32, I32, I32, F, P, I32, P]
    L.mnmt_op_attention_bf16.argtypes = [P, I64, P, I64, I32, I32, P, P, I32, I32, I32, F, P, P, P]
    L.mnmt_op_gather_rows.argtypes = [P, P, P, P, P, I32, P, P, P]
    L.mnmt_op_gemm_i8_split.argtypes = [P, P, I32, I32, I32, P, F, I32, P, P, I32, I32, P]
    L.mnmt_op_src_attention.argtypes = [P, I64, P, I64, I64, I32, I32, P, P, I32, I32, I32, I32, F, P, P, P]
    L.mnmt_op_src_attention_f32.argtypes = [P, I64, P, I64, I64, I32, I32, P, P, I32, I32, I32, I32, F, P, P, P]
    for name in EXPORTS:
        fn = getattr(L, name)
        if name not in ("mnmt_config_default", "mnmt_last_error", "mnmt_model_destroy"):
            fn.restype = S
    _lib = L
    return L


def _check(st: int) -> None:
    if st != 0:
        raise MnmtError(st, lib().mnmt_last_error().decode(errors="replace"))


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def config_from_dims(m) -> Config:
    c = Config()
    c.abi_version = ABI_VERSION
    for f in ("d_model", "d_ffn", "n_heads", "enc_layers", "dec_layers", "vocab", "decoder",
              "aan_ffn_depth", "aan_gate", "out_bias", "eos_id", "clip", "ln_eps"):
        setattr(c, f, getattr(m, f))
    c.src_kv_bf16 = getattr(m, "kv_bf16", 0)
    return c


def batch_by_words(lengths: np.ndarray, budget: int):
    """Length-sorted word-budget batches: (order, batch offsets)."""
    lengths = np.ascontiguousarray(lengths, dtype=np.int32)
    n = int(lengths.shape[0])
    order = np.zeros(max(n, 1), np.int32)
    off = np.zeros(n + 2, np.int32)
    nb = np.zeros(1, np.int32)
    _check(lib().mnmt_batch_by_words(_p(lengths), n, budget, _p(order), _p(off), _p(nb)))
    return order[:n].copy(), off[:nb[0] + 1].copy()


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return int(stream.cuda_stream)   # torch.cuda.Stream


class Model:
    """A student loaded on one GPU: set every parameter, then quantize once."""

    def __init__(self, dims, weights: Optional[Dict[str, np.ndarray]] = None, device: int = 0):
        self.dims = dims
        self.cfg = config_from_dims(dims)
        h = C.c_void_p()
        _check(lib().mnmt_model_create(C.byref(self.cfg), device, C.byref(h)))
        self.h = h
        self.device = device
        if weights is not None:
            for k, v in weights.items():
                self.set_param(k, v)
            self.quantize()

    def set_param(self, name: str, arr: np.ndarray) -> None:
        a = np.ascontiguousarray(arr, dtype=np.float32)
        _check(lib().mnmt_model_set_param(self.h, name.encode(), _p(a), a.size))

    def quantize(self) -> None:
        _check(lib().mnmt_model_quantize(self.h))

    def close(self) -> None:
        if getattr(self, "h", None):
            lib().mnmt_model_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_option(self, name: str, value: int) -> None:
        """Scheduling options (include/mnmt.h); never change results."""
        _check(lib().mnmt_model_set_option(self.h, name.encode(), int(value)))

    def stats(self) -> Dict[str, int]:
        s = Stats()
        _check(lib().mnmt_get_stats(self.h, C.byref(s)))
        return {f: int(getattr(s, f)) for f, _ in Stats._fields_}

    @staticmethod
    def _split(out: np.ndarray, out_len: np.ndarray, max_len: np.ndarray) -> List[np.ndarray]:
        """Per-sentence id arrays: views into `out` (a fresh buffer of this call)."""
        n = len(max_len)
        offs = np.zeros(n + 1, np.int64)
        np.cumsum(max_len, out=offs[1:])
        starts = offs[:-1].tolist()
        ends = (offs[:-1] + out_len[:n]).tolist()
        return [out[a:b] for a, b in zip(starts, ends)]

    def decode(self, sset, stream=None) -> List[np.ndarray]:
        """All sentences of `sset` as one batch, in the given order."""
        n = sset.n
        ml = np.ascontiguousarray(sset.max_len, np.int32)
        out = np.zeros(max(int(ml.sum()), 1), np.int32)
        out_len = np.zeros(max(n, 1), np.int32)
        ids = np.ascontiguousarray(sset.ids, np.int32)
        offs = np.ascontiguousarray(sset.offsets, np.int64)
        _check(lib().mnmt_decode(self.h, _p(ids), _p(offs), n, _p(ml), _p(out), out.size,
                                 _p(out_len), _stream_ptr(stream)))
        return self._split(out, out_len, ml)

    def set_shortlist(self, freq: np.ndarray, lex: np.ndarray) -> None:
        """Shortlist tables (F2): freq [n_freq] ids, lex [vocab x k_lex] ids (include/mnmt.h)."""
        freq = np.ascontiguousarray(freq, np.int32)
        lex = np.ascontiguousarray(lex, np.int32)
        k = lex.shape[1] if lex.ndim == 2 else 0
        _check(lib().mnmt_model_set_shortlist(self.h, _p(freq), freq.size, _p(lex), k))

    def translate(self, sset, budget: int, stream=None, shortlist: bool = False) -> List[np.ndarray]:
        """The whole job (host buffers): batch_by_words + decode of every batch (shortlist:
        each batch's argmax restricted to its vocabulary shortlist, MNMT_SHORTLIST)."""
        n = sset.n
        ml = np.ascontiguousarray(sset.max_len, np.int32)
        out = np.zeros(max(int(ml.sum()), 1), np.int32)
        out_len = np.zeros(max(n, 1), np.int32)
        ids = np.ascontiguousarray(sset.ids, np.int32)
        offs = np.ascontiguousarray(sset.offsets, np.int64)
        _check(lib().mnmt_translate(self.h, _p(ids), _p(offs), n, _p(ml), budget, _p(out),
                                    out.size, _p(out_len), SHORTLIST if shortlist else 0,
                                    _stream_ptr(stream)))
        return self._split(out, out_len, ml)

    def beam_translate(self, sset, budget: int, beam: int, stream=None):
        """Beam search of the whole job (host buffers; include/mnmt.h mnmt_beam_translate).
        Returns, per sentence in input order, [(ids, score)] by descending score."""
        n = sset.n
        ml = np.ascontiguousarray(sset.max_len, np.int32)
        out = np.zeros(max(int(ml.sum()) * beam, 1), np.int32)
        out_len = np.zeros(max(n * beam, 1), np.int32)
        out_score = np.zeros(max(n * beam, 1), np.float32)
        n_hyp = np.zeros(max(n, 1), np.int32)
        ids = np.ascontiguousarray(sset.ids, np.int32)
        offs = np.ascontiguousarray(sset.offsets, np.int64)
        _check(lib().mnmt_beam_translate(self.h, _p(ids), _p(offs), n, _p(ml), budget, beam,
                                         _p(out), out.size, _p(out_len), _p(out_score), _p(n_hyp),
                                         0, _stream_ptr(stream)))
        res, o = [], 0
        for i in range(n):
            T = int(ml[i])
            res.append([(out[beam * o + r * T: beam * o + r * T + out_len[i * beam + r]].copy(),
                         float(out_score[i * beam + r])) for r in range(n_hyp[i])])
            o += T
        return res

    def beam_translate_device(self, ids_ptr: int, offsets: np.ndarray, max_len: np.ndarray,
                              budget: int, beam: int, out_ptr: int, out_cap: int,
                              out_len_ptr: int, out_score_ptr: int, n_hyp_ptr: int,
                              stream=None) -> None:
        """Beam search with ids and outputs resident in HBM (MNMT_DEVICE_IO)."""
        offs = np.ascontiguousarray(offsets, np.int64)
        ml = np.ascontiguousarray(max_len, np.int32)
        _check(lib().mnmt_beam_translate(self.h, ids_ptr, _p(offs), len(ml), _p(ml), budget, beam,
                                         out_ptr, out_cap, out_len_ptr, out_score_ptr, n_hyp_ptr,
                                         DEVICE_IO, _stream_ptr(stream)))

    def translate_device(self, ids_ptr: int, offsets: np.ndarray, max_len: np.ndarray,
                         budget: int, out_ptr: int, out_cap: int, out_len_ptr: int,
                         stream=None, shortlist: bool = False) -> None:
        """The whole job with ids already resident in HBM (MNMT_DEVICE_IO)."""
        offs = np.ascontiguousarray(offsets, np.int64)
        ml = np.ascontiguousarray(max_len, np.int32)
        _check(lib().mnmt_translate(self.h, ids_ptr, _p(offs), len(ml), _p(ml), budget, out_ptr,
                                    out_cap, out_len_ptr, DEVICE_IO | (SHORTLIST if shortlist else 0),
                                    _stream_ptr(stream)))

    def decode_forced(self, sset, forced: np.ndarray, forced_off: np.ndarray,
                      dump_mask: int = 0, stream=None, budget: Optional[int] = None):
        """Teacher forcing (P-2): returns (argmax ids flat [sum T_i], dumps dict).
        budget None: all sentences as one batch (mnmt_decode_forced); otherwise the whole
        translate schedule (word-budget batches, waves, lanes, step graphs) with that budget
        (mnmt_translate_forced; encoder dumps unavailable)."""
        n = sset.n
        d, L = self.dims.d_model, self.dims.dec_layers
        ids = np.ascontiguousarray(sset.ids, np.int32)
        offs = np.ascontiguousarray(sset.offsets, np.int64)
        f = np.ascontiguousarray(forced, np.int32)
        fo = np.ascontiguousarray(forced_off, np.int64)
        ntok, O = int(offs[-1]), int(fo[-1])
        sections = []
        if dump_mask & DUMP_ENC_OUT:
            sections.append(("enc_out", np.float32, (ntok, d)))
        if dump_mask & DUMP_SRC_KV:
            sections.append(("src_kv", np.float32, (L, ntok, 2, d)))
        if dump_mask & DUMP_DEC_OUT:
            sections.append(("dec_out", np.float32, (O, d)))
        if dump_mask & DUMP_OUT_CODES:
            sections.append(("out_codes", np.int8, (O, d)))
        if dump_mask & DUMP_LAYERS:
            sections.append(("layers", np.float32, (O, L, 3, d)))
        if dump_mask & DUMP_MARGIN:
            sections.append(("margin", np.float32, (O,)))
        nbytes = sum(int(np.prod(s)) * np.dtype(t).itemsize for _, t, s in sections)
        buf = np.zeros(max(nbytes, 1), np.uint8)
        am = np.zeros(max(O, 1), np.int32)
        if budget is None:
            _check(lib().mnmt_decode_forced(self.h, _p(ids), _p(offs), n, _p(f if f.size else None),
                                            _p(fo), _p(am), dump_mask, _p(buf), nbytes,
                                            _stream_ptr(stream)))
        else:
            _check(lib().mnmt_translate_forced(self.h, _p(ids), _p(offs), n,
                                               _p(f if f.size else None), _p(fo), int(budget),
                                               _p(am), dump_mask, _p(buf), nbytes,
                                               _stream_ptr(stream)))
        dumps, o = {}, 0
        for name, t, shape in sections:
            k = int(np.prod(shape)) * np.dtype(t).itemsize
            dumps[name] = buf[o:o + k].view(t).reshape(shape).copy()
            o += k
        return am[:O].copy(), dumps


# ---------------------------------------------------------------- op-level entry points
# Pointers are device addresses (e.g. torch_tensor.data_ptr()); stream = torch stream or int.
def op_quantize(x_ptr: int, n: int, clip: float, out_ptr: int, stream=None) -> None:
    _check(lib().mnmt_op_quantize(x_ptr, n, clip, out_ptr, _stream_ptr(stream)))


def op_gemm_i8(A_ptr, W_ptr, M, N, K, bias_ptr, clip, epi, out_ptr, out2_ptr=None, n_tile=0,
               stream=None) -> None:
    _check(lib().mnmt_op_gemm_i8(A_ptr, W_ptr, M, N, K, bias_ptr, clip, epi, out_ptr, out2_ptr,
                                 n_tile, _stream_ptr(stream)))


def op_gemm_i8_split(A_ptr, W_ptr, M, N, K, bias_ptr, clip, epi, out_ptr, out2_ptr=None, n_tile=0,
                     split_k=-1, stream=None) -> None:
    _check(lib().mnmt_op_gemm_i8_split(A_ptr, W_ptr, M, N, K, bias_ptr, clip, epi, out_ptr, out2_ptr,
                                       n_tile, split_k, _stream_ptr(stream)))


def op_attention_enc(qkv_ptr, start_ptr, len_ptr, n_sent, d, H, s_max, clip, out_q_ptr, variant=0,
                     stream=None) -> None:
    _check(lib().mnmt_op_attention_enc(qkv_ptr, start_ptr, len_ptr, n_sent, d, H, s_max, clip,
                                       out_q_ptr, variant, _stream_ptr(stream)))


def op_argmax_ids(keys_ptr, n, ids_ptr, stream=None) -> None:
    _check(lib().mnmt_op_argmax_ids(keys_ptr, n, ids_ptr, _stream_ptr(stream)))


def op_layernorm(x_ptr, delta_ptr, gi_ptr, gf_ptr, gamma_ptr, beta_ptr, n, d, eps, clip,
                 out_ptr, out_q_ptr, stream=None) -> None:
    _check(lib().mnmt_op_layernorm(x_ptr, delta_ptr, gi_ptr, gf_ptr, gamma_ptr, beta_ptr, n, d,
                                   eps, clip, out_ptr, out_q_ptr, _stream_ptr(stream)))


def op_aan_step(C_ptr, y_ptr, n, d, t, clip, g_ptr, g_q_ptr, stream=None) -> None:
    _check(lib().mnmt_op_aan_step(C_ptr, y_ptr, n, d, t, clip, g_ptr, g_q_ptr,
                                  _stream_ptr(stream)))


def op_embed(E_ptr, d, ids_ptr, pos_ptr, n, clip, x_ptr, xq_ptr, stream=None) -> None:
    _check(lib().mnmt_op_embed(E_ptr, d, ids_ptr, pos_ptr, n, clip, x_ptr, xq_ptr,
                               _stream_ptr(stream)))


def op_attention(q_ptr, ldq, kv_ptr, ldkv, k_off, v_off, start_ptr, len_ptr, n, d, H, clip,
                 out_q_ptr, out_f_ptr=None, stream=None) -> None:
    _check(lib().mnmt_op_attention(q_ptr, ldq, kv_ptr, ldkv, k_off, v_off, start_ptr, len_ptr, n,
                                   d, H, clip, out_q_ptr, out_f_ptr, _stream_ptr(stream)))


def op_src_attention_f32(q_ptr, ldq, kv_ptr, kv_rows, ldkv, k_off, v_off, start_ptr, len_ptr,
                         max_span, n, d, H, clip, out_q_ptr, out_f_ptr=None, stream=None) -> None:
    """A7 through the one-warp TMA kernel in fp32 arithmetic (option attn_f32; departs from R20)."""
    _check(lib().mnmt_op_src_attention_f32(q_ptr, ldq, kv_ptr, kv_rows, ldkv, k_off, v_off, start_ptr,
                                           len_ptr, max_span, n, d, H, clip, out_q_ptr, out_f_ptr,
                                           _stream_ptr(stream)))


def op_src_attention(q_ptr, ldq, kv_ptr, kv_rows, ldkv, k_off, v_off, start_ptr, len_ptr,
                     max_span, n, d, H, clip, out_q_ptr, out_f_ptr=None, stream=None) -> None:
    """A7 with the decode path's kernel choice (TMA-tiled for fp32 K/V, d/H = 32 / 64)."""
    _check(lib().mnmt_op_src_attention(q_ptr, ldq, kv_ptr, kv_rows, ldkv, k_off, v_off, start_ptr,
                                       len_ptr, max_span, n, d, H, clip, out_q_ptr, out_f_ptr,
                                       _stream_ptr(stream)))


def op_attention_bf16(q_ptr, ldq, kv16_ptr, ldkv, k_off, v_off, start_ptr, len_ptr, n, d, H, clip,
                      out_q_ptr, out_f_ptr=None, stream=None) -> None:
    _check(lib().mnmt_op_attention_bf16(q_ptr, ldq, kv16_ptr, ldkv, k_off, v_off, start_ptr,
                                        len_ptr, n, d, H, clip, out_q_ptr, out_f_ptr,
                                        _stream_ptr(stream)))


def op_gather_rows(src_ptr, src_off_ptr, src_len_ptr, dst_row_ptr, dst_off_ptr, n, dst_ptr,
                   dst_len_ptr, stream=None) -> None:
    """A11 on several GPUs: gathered rows back to input order (include/mnmt_ops.h)."""
    _check(lib().mnmt_op_gather_rows(src_ptr, src_off_ptr, src_len_ptr, dst_row_ptr, dst_off_ptr,
                                     n, dst_ptr, dst_len_ptr, _stream_ptr(stream)))
