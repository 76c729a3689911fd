"""Independent numpy reference in the TRAINING-TIME (parallel) form.

Used only to pin the oracle (tests/test_oracle_pins.py).  It differs from the
oracle in formulation, not just in language:
  * the AAN average is the whole-sequence cumulative form G = cumsum(Y)/t over
    the time axis ("cumulative uniform averaging operation across
    the previous layer"), not the oracle's carried running-sum state;
  * decoder self-attention is one causally-masked attention over all positions
    (PAPER.md:L71), not an incremental KV cache;
  * integer products are numpy int64 matrix products, LayerNorm/attention are
    vectorised float64 numpy.
Quantisation follows the same fixed rule (R1, R2).
Runs teacher-forced: inputs[0] is the start symbol, inputs[t] = forced[t-1].
"""
from __future__ import annotations

import math

import numpy as np


def q8(x, clip=2.0):
    x = np.asarray(x, np.float32)
    sig = np.float32(127.0) / np.float32(clip)
    return np.rint(np.clip(x, np.float32(-clip), np.float32(clip)) * sig).astype(np.int8)


def bf16_round(x):
    """Nearest bfloat16 (ties to even) by arithmetic, not bit patterns: a normal value keeps 8
    significant bits (frexp mantissa in [0.5, 1) scaled by 2^8, rint = half-even); below
    2^-126 the bfloat16 grid is the fixed subnormal step 2^-133."""
    x = np.asarray(x, np.float64)
    m, e = np.frexp(x)
    normal = np.ldexp(np.rint(np.ldexp(m, 8)), e - 8)
    sub = np.rint(np.ldexp(x, 133)) * 2.0 ** -133
    return np.where(np.abs(x) < 2.0 ** -126, sub, normal).astype(np.float32)


def dq_scale(clip=2.0):
    return np.float32(clip * clip / (127.0 * 127.0))


def lin(codes, Wq, b, s):
    """fmaf((float)acc, s, b): acc*s is exact in float64 (<= 48 significant bits)."""
    acc = codes.astype(np.int64) @ Wq.astype(np.int64).T
    v = acc.astype(np.float64) * np.float64(s)
    if b is not None:
        v = v + b.astype(np.float64)
    return v.astype(np.float32), acc


def layernorm(r, g, b, eps):
    r64 = r.astype(np.float64)
    mu = r64.mean(axis=-1, keepdims=True)
    var = ((r64 - mu) ** 2).mean(axis=-1, keepdims=True)
    return ((r64 - mu) / np.sqrt(var + np.float64(np.float32(eps))) * g.astype(np.float64)
            + b.astype(np.float64)).astype(np.float32)


def attention(Q, K, V, H, causal=False):
    """Q [Tq x d], K/V [Tk x d]; fp64, softmax with max subtraction."""
    Tq, d = Q.shape
    dh = d // H
    out = np.empty((Tq, d), np.float32)
    for h in range(H):
        q = Q[:, h * dh:(h + 1) * dh].astype(np.float64)
        k = K[:, h * dh:(h + 1) * dh].astype(np.float64)
        v = V[:, h * dh:(h + 1) * dh].astype(np.float64)
        sc = (q @ k.T) * (1.0 / math.sqrt(dh))
        if causal:
            sc = np.where(np.tril(np.ones_like(sc, dtype=bool)), sc, -np.inf)
        sc = sc - sc.max(axis=1, keepdims=True)
        p = np.exp(sc)
        out[:, h * dh:(h + 1) * dh] = ((p @ v) / p.sum(axis=1, keepdims=True)).astype(np.float32)
    return out


def pe_table(T, d):
    P = np.zeros((T, d), np.float32)
    for pos in range(T):
        for i in range(0, d, 2):
            ang = pos / math.pow(10000.0, i / d)
            P[pos, i] = np.float32(math.sin(ang))
            if i + 1 < d:
                P[pos, i + 1] = np.float32(math.cos(ang))
    return P


def embed(E, ids, pos0, d):
    r = np.float32(math.sqrt(d))
    P = pe_table(pos0 + len(ids), d)[pos0:]
    e = np.zeros((len(ids), d), np.float32)
    for i, t in enumerate(ids):
        if t >= 0:
            e[i] = E[t] * r
    return e + P


def sigmoid(x):
    return (1.0 / (1.0 + np.exp(-x.astype(np.float64)))).astype(np.float32)


class ParallelModel:
    def __init__(self, dims, w):
        self.m = dims
        self.w = w
        c = dims.clip
        self.s = dq_scale(c)
        self.qw = {k: q8(v, c) for k, v in w.items() if k.endswith(".W") or k == "emb.E"}

    def L(self, name, codes):
        return lin(codes, self.qw[name + ".W"], self.w[name + ".b"], self.s)[0]

    def encode(self, src):
        m, w = self.m, self.w
        d, c = m.d_model, m.clip
        x = embed(w["emb.E"], list(src), 0, d)
        for l in range(m.enc_layers):
            p = f"enc.{l}."
            qx = q8(x, c)
            Q, K, V = (self.L(p + f"self.{n}", qx) for n in "qkv")
            ctx = attention(Q, K, V, m.n_heads)
            x = layernorm(x + self.L(p + "self.o", q8(ctx, c)), w[p + "ln1.g"], w[p + "ln1.b"], m.ln_eps)
            h = q8(np.maximum(self.L(p + "ffn.1", q8(x, c)), np.float32(0)), c)
            x = layernorm(x + self.L(p + "ffn.2", h), w[p + "ln2.g"], w[p + "ln2.b"], m.ln_eps)
        qx = q8(x, c)
        kv = np.stack([np.stack([self.L(f"dec.{l}.src.k", qx), self.L(f"dec.{l}.src.v", qx)])
                       for l in range(m.dec_layers)])
        if getattr(m, "kv_bf16", 0):
            kv = bf16_round(kv)
        return x, kv

    def forced(self, src, forced, T):
        """All T steps at once; returns ids [T], dec_out [T x d], logits [T x V]."""
        m, w = self.m, self.w
        d, c = m.d_model, m.clip
        _, kv = self.encode(src)
        inputs = [-1] + list(forced[:T - 1])
        y = embed(w["emb.E"], inputs, 0, d)
        t = np.arange(1, T + 1, dtype=np.float32)[:, None]
        for l in range(m.dec_layers):
            p = f"dec.{l}."
            if m.decoder == 1:
                G = np.cumsum(y, axis=0, dtype=np.float32) / t      # cumulative average
                if m.aan_ffn_depth == 0:
                    a = G
                elif m.aan_ffn_depth == 1:
                    a = np.maximum(self.L(p + "aan.ffn.1", q8(G, c)), np.float32(0))
                else:
                    h = q8(np.maximum(self.L(p + "aan.ffn.1", q8(G, c)), np.float32(0)), c)
                    a = self.L(p + "aan.ffn.2", h)
                if m.aan_gate:
                    gi = sigmoid(self.L(p + "aan.gate.i", q8(y, c)))
                    gf = sigmoid(self.L(p + "aan.gate.f", q8(a, c)))
                    z = gi * y + gf * a
                else:
                    z = a
            else:
                qy = q8(y, c)
                Q, K, V = (self.L(p + f"self.{n}", qy) for n in "qkv")
                z = self.L(p + "self.o", q8(attention(Q, K, V, m.n_heads, causal=True), c))
            x1 = layernorm(y + z, w[p + "ln1.g"], w[p + "ln1.b"], m.ln_eps)
            qs = self.L(p + "src.q", q8(x1, c))
            ctx = attention(qs, kv[l, 0], kv[l, 1], m.n_heads)
            x2 = layernorm(x1 + self.L(p + "src.o", q8(ctx, c)), w[p + "ln2.g"], w[p + "ln2.b"], m.ln_eps)
            h = q8(np.maximum(self.L(p + "ffn.1", q8(x2, c)), np.float32(0)), c)
            y = layernorm(x2 + self.L(p + "ffn.2", h), w[p + "ln3.g"], w[p + "ln3.b"], m.ln_eps)
        logits, _ = lin(q8(y, c), self.qw["emb.E"], w.get("out.b"), self.s)
        ids = np.argmax(logits, axis=1)          # first maximum = lowest id
        return ids.astype(np.int32), y, logits
