"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic: it only draws random
numbers (weights, sentence lengths, token ids) and names parameters.  Both
`oracle/` and `paper_1805_12096_b200/` receive the arrays it returns; neither
imports the other.

Model dimensions: PAPER.md:L49-63 (Table 1 `trans.dim`), 36,000 joint BPE
vocabulary with tied embeddings, six blocks per stack
(PAPER.md:L65), AAN with FFN width = embedding size.
Sentence-set shape: newstest2014 = 3003 sentences, 62,954 source tokens
(PAPER.md:L475), lengths log-normal (SURVEY.md 8(d) "Synthetic inputs").
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List

import numpy as np

EOS_ID, UNK_ID, PAD_ID = 0, 1, 2          # reserved ids (SPEC.md:L497 reading)
VOCAB = 36000
NEWSTEST_SENTENCES = 3003                 # BASELINE.json configs[1]
NEWSTEST_TOKENS = 62954


@dataclasses.dataclass(frozen=True)
class ModelDims:
    """Dimensions of a student (Table 1)."""
    name: str
    d_model: int
    d_ffn: int
    n_heads: int
    decoder: int = 1            # 1 = AAN, 0 = self-attention + KV cache
    aan_ffn_depth: int = 2      # 0 = "-ffn", 1, 2 (reading R9)
    aan_gate: int = 1           # 0 = "-gate"
    enc_layers: int = 6
    dec_layers: int = 6
    vocab: int = VOCAB
    out_bias: int = 1
    eos_id: int = EOS_ID
    clip: float = 2.0
    ln_eps: float = 1e-6        # DESIGN.md reading R10
    kv_bf16: int = 0            # 1: source K/V rounded to bf16 (R35)


PRESETS: Dict[str, ModelDims] = {
    "tiny192-aan": ModelDims("tiny192-aan", 192, 1536, 8),
    "tiny192-aan-noffn-nogate": ModelDims("tiny192-aan-noffn-nogate", 192, 1536, 8,
                                          aan_ffn_depth=0, aan_gate=0),
    "small-aan": ModelDims("small-aan", 256, 2048, 8),
    "small-aan-noffn": ModelDims("small-aan-noffn", 256, 2048, 8, aan_ffn_depth=0),
    "small": ModelDims("small", 256, 2048, 8, decoder=0),
    "base-aan": ModelDims("base-aan", 512, 2048, 8),
    "base": ModelDims("base", 512, 2048, 8, decoder=0),
    "big": ModelDims("big", 1024, 4096, 16, decoder=0),
}


def param_shapes(m: ModelDims) -> Dict[str, tuple]:
    """Parameter manifest (include/mnmt.h "Parameter manifest").

    Every W is row-major [out x in]: the B^T operand of dotint(A, B)
    (PAPER.md:L100)."""
    d, F = m.d_model, m.d_ffn
    s: Dict[str, tuple] = {"emb.E": (m.vocab, d)}
    if m.out_bias:
        s["out.b"] = (m.vocab,)

    def lin(prefix, out, inp):
        s[prefix + ".W"] = (out, inp)
        s[prefix + ".b"] = (out,)

    def ln(prefix):
        s[prefix + ".g"] = (d,)
        s[prefix + ".b"] = (d,)

    for l in range(m.enc_layers):
        for p in "qkvo":
            lin(f"enc.{l}.self.{p}", d, d)
        lin(f"enc.{l}.ffn.1", F, d)
        lin(f"enc.{l}.ffn.2", d, F)
        ln(f"enc.{l}.ln1")
        ln(f"enc.{l}.ln2")
    for l in range(m.dec_layers):
        if m.decoder == 1:
            if m.aan_ffn_depth >= 1:
                lin(f"dec.{l}.aan.ffn.1", d, d)
            if m.aan_ffn_depth >= 2:
                lin(f"dec.{l}.aan.ffn.2", d, d)
            if m.aan_gate:
                lin(f"dec.{l}.aan.gate.i", d, d)
                lin(f"dec.{l}.aan.gate.f", d, d)
        else:
            for p in "qkvo":
                lin(f"dec.{l}.self.{p}", d, d)
        for p in "qkvo":
            lin(f"dec.{l}.src.{p}", d, d)
        lin(f"dec.{l}.ffn.1", F, d)
        lin(f"dec.{l}.ffn.2", d, F)
        ln(f"dec.{l}.ln1")
        ln(f"dec.{l}.ln2")
        ln(f"dec.{l}.ln3")
    return s


def make_weights(m: ModelDims, seed: int = 1, code_domain: bool = False,
                 emb_scale: float = 0.5) -> Dict[str, np.ndarray]:
    """Random-init weights (SURVEY.md 8(d) "Synthetic inputs").

    Linear W ~ Glorot-uniform +-sqrt(6/(in+out)); E ~ U(-0.5, 0.5); biases
    U(-0.1, 0.1); LN gain 1 + U(-0.1, 0.1), LN bias U(-0.1, 0.1).
    code_domain=True draws every W (and E) as k/63.5, k uniform in [-127,127]
    (GEMM stress: every code is reachable).  emb_scale sets E ~ U(-emb_scale, emb_scale);
    a small scale weakens the tied-embedding feedback so free-running outputs vary."""
    rng = np.random.default_rng(seed)
    out: Dict[str, np.ndarray] = {}
    for name, shape in param_shapes(m).items():
        if name == "emb.E":
            if code_domain:
                a = rng.integers(-127, 128, size=shape).astype(np.float32) / np.float32(63.5)
            else:
                a = rng.uniform(-emb_scale, emb_scale, size=shape)
        elif name.endswith(".W"):
            if code_domain:
                a = rng.integers(-127, 128, size=shape).astype(np.float32) / np.float32(63.5)
            else:
                bound = np.sqrt(6.0 / (shape[0] + shape[1]))
                a = rng.uniform(-bound, bound, size=shape)
        elif name.endswith(".g"):
            a = 1.0 + rng.uniform(-0.1, 0.1, size=shape)
        else:  # biases, LN beta, out.b
            a = rng.uniform(-0.1, 0.1, size=shape)
        out[name] = np.ascontiguousarray(a, dtype=np.float32)
    return out


@dataclasses.dataclass
class SentenceSet:
    """Source sentences as a flat id array plus offsets (include/mnmt.h)."""
    ids: np.ndarray        # int32 [sum S_i]
    offsets: np.ndarray    # int64 [n+1]
    max_len: np.ndarray    # int32 [n]  (= S_i; reading R16)

    @property
    def n(self) -> int:
        return int(self.offsets.shape[0] - 1)

    @property
    def lengths(self) -> np.ndarray:
        return np.diff(self.offsets).astype(np.int32)

    def subset(self, idx) -> "SentenceSet":
        idx = np.asarray(idx, dtype=np.int64)
        lens = self.lengths[idx]
        offs = np.zeros(len(idx) + 1, dtype=np.int64)
        offs[1:] = np.cumsum(lens)
        ids = np.concatenate([self.ids[self.offsets[i]:self.offsets[i + 1]] for i in idx]) \
            if len(idx) else np.zeros(0, np.int32)
        return SentenceSet(ids.astype(np.int32), offs, self.max_len[idx].copy())


def _from_lengths(lengths: np.ndarray, rng, vocab: int) -> SentenceSet:
    lengths = np.asarray(lengths, dtype=np.int64)
    offs = np.zeros(len(lengths) + 1, dtype=np.int64)
    offs[1:] = np.cumsum(lengths)
    ids = rng.integers(3, vocab, size=int(offs[-1]), dtype=np.int64).astype(np.int32)
    return SentenceSet(ids, offs, lengths.astype(np.int32))


def newstest_lengths(seed: int = 2014, n: int = NEWSTEST_SENTENCES, total: int = NEWSTEST_TOKENS,
                     sigma: float = 0.55, lo: int = 1, hi: int = 100) -> np.ndarray:
    """newstest2014-shaped lengths: RNE(lognormal), clipped to [lo, hi], then
    nudged +-1 at random rows until the sum is exactly `total`."""
    rng = np.random.default_rng(seed)
    mean = total / n
    mu = np.log(mean) - sigma * sigma / 2
    L = np.clip(np.rint(rng.lognormal(mu, sigma, size=n)), lo, hi).astype(np.int64)
    diff = int(total - L.sum())
    while diff != 0:
        i = int(rng.integers(0, n))
        step = 1 if diff > 0 else -1
        if lo <= L[i] + step <= hi:
            L[i] += step
            diff -= step
    return L


def newstest_set(seed: int = 2014, vocab: int = VOCAB, n: int = NEWSTEST_SENTENCES,
                 total: int = NEWSTEST_TOKENS) -> SentenceSet:
    L = newstest_lengths(seed, n, total)
    return _from_lengths(L, np.random.default_rng(seed + 1), vocab)


def uniform_set(n: int, length: int, seed: int = 7, vocab: int = VOCAB) -> SentenceSet:
    """n sentences of one length (configs[0]: 4 x 20; configs[4] sweeps)."""
    return _from_lengths(np.full(n, length), np.random.default_rng(seed), vocab)


def random_set(n: int, lo: int, hi: int, seed: int = 11, vocab: int = VOCAB) -> SentenceSet:
    rng = np.random.default_rng(seed)
    L = rng.integers(lo, hi + 1, size=n)
    return _from_lengths(L, rng, vocab)


def forced_targets(lengths: List[int], seed: int = 5, vocab: int = VOCAB) -> np.ndarray:
    """Teacher-forcing prefixes: random non-reserved ids, flat [sum T_i]."""
    rng = np.random.default_rng(seed)
    return rng.integers(3, vocab, size=int(np.sum(lengths)), dtype=np.int64).astype(np.int32)


def uniform_activations(shape, seed: int = 3, scale: float = 2.5) -> np.ndarray:
    """Generic fp32 operand for kernel-level parity (values beyond +-clip included)."""
    rng = np.random.default_rng(seed)
    return rng.uniform(-scale, scale, size=shape).astype(np.float32)


def shortlist_tables(vocab: int = VOCAB, n_freq: int = 100, k_lex: int = 100, seed: int = 85,
                     zipf: float = 1.1):
    """Synthetic lexical shortlist tables (SPEC.md:L497 format):
    `freq` = the n_freq most frequent target ids (a seeded frequency ranking of the vocabulary),
    `lex` [vocab x k_lex] = for every source id, k_lex distinct target ids in descending
    translation probability, drawn from a Zipf(zipf) law over the frequency ranking (frequent
    words are likely translations of many source words, so batch unions overlap).  Random
    numbers only; the union itself is the method's and lives in oracle/ and the CUDA path."""
    rng = np.random.default_rng(seed)
    rank = rng.permutation(vocab).astype(np.int32)         # rank[r] = id of the r-th most frequent
    cdf = np.cumsum(1.0 / np.arange(1, vocab + 1, dtype=np.float64) ** zipf)
    cdf /= cdf[-1]
    draws = np.minimum(np.searchsorted(cdf, rng.random((vocab, 3 * k_lex))), vocab - 1)
    lex = np.empty((vocab, k_lex), np.int32)
    for s in range(vocab):
        _, first = np.unique(draws[s], return_index=True)
        r = draws[s][np.sort(first)][:k_lex]               # distinct ranks in draw order
        if r.size < k_lex:                                 # top up with uniform distinct ranks
            extra = rng.permutation(np.setdiff1d(np.arange(vocab), r))[:k_lex - r.size]
            r = np.concatenate([r, extra])
        lex[s] = rank[r]
    return rank[:n_freq].copy(), lex


# ---------------------------------------------------------------- files for the C client
# (examples/mnmt_translate.c): plain binary records, little-endian.
def write_weights_bin(path: str, m: ModelDims, weights: Dict[str, np.ndarray]) -> None:
    """{int32 name_len, name, int64 numel, float32[numel]} for every parameter of the manifest."""
    with open(path, "wb") as f:
        for name in param_shapes(m):
            a = np.ascontiguousarray(weights[name], np.float32).ravel()
            b = name.encode()
            f.write(np.int32(len(b)).tobytes() + b + np.int64(a.size).tobytes() + a.tobytes())


def write_sentences_bin(path: str, sset: "SentenceSet") -> None:
    """{int32 n, int64 offsets[n+1], int32 ids[offsets[n]], int32 max_len[n]}."""
    with open(path, "wb") as f:
        f.write(np.int32(sset.n).tobytes() + np.ascontiguousarray(sset.offsets, np.int64).tobytes()
                + np.ascontiguousarray(sset.ids, np.int32).tobytes()
                + np.ascontiguousarray(sset.max_len, np.int32).tobytes())


def write_shortlist_bin(path: str, freq: np.ndarray, lex: np.ndarray) -> None:
    """{int32 n_freq, int32 freq[n_freq], int32 k_lex, int32 lex[vocab * k_lex]}."""
    freq = np.ascontiguousarray(freq, np.int32)
    lex = np.ascontiguousarray(lex, np.int32)
    with open(path, "wb") as f:
        f.write(np.int32(freq.size).tobytes() + freq.tobytes() + np.int32(lex.shape[1]).tobytes()
                + lex.tobytes())

