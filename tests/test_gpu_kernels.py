"""P-1: kernel parity with injected operands.  Every CUDA kernel gets the
oracle's exact inputs through the op-level C-ABI (include/mnmt_ops.h) and is compared with
the oracle: s32 accumulators, fmaf epilogues, codes and argmax bit-exactly; fp64-reduced
floats (LN, attention) exactly up to rare last-bit double-rounding events."""
import numpy as np
import pytest

import oracle.oracle as O
import synth
from tests.gpu_util import boundary_explained, empty, ptr, sync, to_dev, torch_dev, zeros

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1805_12096_b200 import mnmt as M  # noqa: E402

CLIP = 2.0


def rand_codes(shape, seed):
    return np.random.default_rng(seed).integers(-127, 128, size=shape).astype(np.int8)


# ------------------------------------------------------------------ quantizer (A1)
def test_quantize_bitexact():
    x = synth.uniform_activations((1 << 20,), seed=1, scale=3.0)
    # add every exact half case k + 1/2 (R1) and the clip boundaries
    halves = []
    for k in range(-127, 127):
        x0 = np.float32((k + 0.5) / 63.5)
        for _ in range(3):
            if np.float32(x0) * np.float32(63.5) == np.float32(k + 0.5):
                halves.append(x0)
            x0 = np.nextafter(x0, np.float32(np.inf), dtype=np.float32)
    x = np.concatenate([x, np.array(halves, np.float32), np.array([2.0, -2.0, 0.0, -0.0, 1e9, -1e9], np.float32)])
    xd = to_dev(x)
    out = empty((x.size,), torch.int8)
    M.op_quantize(ptr(xd), x.size, CLIP, ptr(out))
    sync()
    assert np.array_equal(out.cpu().numpy(), O.quantize(x, CLIP))


# ------------------------------------------------------------------ int8 GEMM (A3, A4, A6-A9)
GEMM_SHAPES = [
    (1, 64, 64, 0), (4, 192, 192, 64), (130, 256, 192, 64), (300, 2048, 256, 128),
    (257, 1536, 2048, 256), (383, 512, 1024, 0), (128, 6144, 512, 256), (77, 36000, 256, 256),
    (520, 256, 2048, 128), (1000, 1024, 4096, 0),
    (5000, 2048, 256, 0), (4999, 768, 512, 256),      # > 2 waves of tiles: persistent kernel
]


@pytest.mark.parametrize("Mr,N,K,bn", GEMM_SHAPES)
def test_gemm_acc_bitexact(Mr, N, K, bn):
    a = rand_codes((Mr, K), Mr + K)
    w = rand_codes((N, K), N + 7)
    out = empty((Mr, N), torch.int32)
    M.op_gemm_i8(ptr(to_dev(a)), ptr(to_dev(w)), Mr, N, K, None, CLIP, M.EPI_ACC, ptr(out), None, bn)
    sync()
    assert np.array_equal(out.cpu().numpy(), O.gemm_acc(a, w))


# split-K (mnmt_op_gemm_i8_split): the K blocks of one output tile are spread over a cluster of
# 2 / 4 / 8 CTAs whose s32 partials are added in the leader's shared memory
SPLIT_K_SHAPES = [
    (1, 1024, 1024, 64, 4),      # one K range of 2 blocks per CTA
    (128, 1024, 4096, 64, 4),    # 8 K blocks each
    (100, 3072, 1024, 0, 2),
    (200, 1024, 2048, 128, 2),   # 2 M tiles, BN 128
    (37, 4096, 1024, 0, -1),     # the library's rule (no split here)
    (32, 1024, 4096, 64, -1),    # the rule: 4 CTAs
    (70, 1024, 1040, 64, 4),     # ragged K: 9 blocks -> fewer, non-empty ranges
    (257, 1024, 1024, 64, 8),    # three M tiles, a ragged one; 8 -> capped by shared memory
    (5, 256, 256, 64, 2),        # two K blocks, one each
]


@pytest.mark.parametrize("Mr,N,K,bn,ks", SPLIT_K_SHAPES)
def test_gemm_split_k_acc_bitexact(Mr, N, K, bn, ks):
    a = rand_codes((Mr, K), Mr + K + 1)
    w = rand_codes((N, K), N + 9)
    out = empty((Mr, N), torch.int32)
    M.op_gemm_i8_split(ptr(to_dev(a)), ptr(to_dev(w)), Mr, N, K, None, CLIP, M.EPI_ACC, ptr(out), None, bn, ks)
    sync()
    assert np.array_equal(out.cpu().numpy(), O.gemm_acc(a, w))


@pytest.mark.parametrize("epi", [M.EPI_F32, M.EPI_F32_Q, M.EPI_RELU_Q, M.EPI_RELU_F32_Q, M.EPI_SIGMOID])
@pytest.mark.parametrize("Mr,N,K", [(5, 256, 256), (33, 1024, 1024), (120, 1024, 4096), (260, 2048, 512), (131, 512, 2048),
                                    (70, 160, 256), (1, 32, 64),   # 32-wide tiles, ragged N
                                    (4700, 2048, 256)])   # last: persistent kernel
def test_gemm_epilogues_bitexact(epi, Mr, N, K):
    rng = np.random.default_rng(epi * 100 + Mr)
    x = rng.normal(0, 1.0, size=(Mr, K)).astype(np.float32)
    W = rng.uniform(-0.08, 0.08, size=(N, K)).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, size=N).astype(np.float32)
    qa, qw = O.quantize(x), O.quantize(W)
    v = O.linear(qa, qw, b, CLIP)                                   # oracle: fmaf((float)acc, s, b)
    A, Wd, bd = to_dev(qa), to_dev(qw), to_dev(b)
    of = empty((Mr, N), torch.float32)
    oq = empty((Mr, N), torch.int8)
    ks = 4 if K >= 1024 else 1      # deep K: through a split-K cluster
    if epi == M.EPI_RELU_Q:
        M.op_gemm_i8_split(ptr(A), ptr(Wd), Mr, N, K, ptr(bd), CLIP, epi, ptr(oq), None, 0, ks)
    else:
        M.op_gemm_i8_split(ptr(A), ptr(Wd), Mr, N, K, ptr(bd), CLIP, epi, ptr(of), ptr(oq), 0, ks)
    sync()
    if epi == M.EPI_F32:
        assert np.array_equal(of.cpu().numpy(), v)
    elif epi == M.EPI_F32_Q:
        assert np.array_equal(of.cpu().numpy(), v)
        assert np.array_equal(oq.cpu().numpy(), O.quantize(v))
    elif epi == M.EPI_RELU_Q:
        assert np.array_equal(oq.cpu().numpy(), O.quantize(np.maximum(v, np.float32(0))))
    elif epi == M.EPI_RELU_F32_Q:
        r = np.maximum(v, np.float32(0))
        assert np.array_equal(of.cpu().numpy(), r)
        assert np.array_equal(oq.cpu().numpy(), O.quantize(r))
    else:
        assert np.array_equal(of.cpu().numpy(), O.sigmoid_array(v))


@pytest.mark.parametrize("epi", [M.EPI_F32, M.EPI_F32_Q, M.EPI_RELU_Q, M.EPI_RELU_F32_Q, M.EPI_SIGMOID])
@pytest.mark.parametrize("Mr,N,K,bias", [(1, 256, 256, True), (7, 2048, 256, True), (32, 256, 2048, True),
                                         (32, 512, 512, False), (19, 48, 96, True), (32, 16, 16, True),
                                         (13, 1024, 4096, True), (32, 208, 192, True)])
def test_gemm_small_m_bitexact(epi, Mr, N, K, bias):
    """k_gemm_smallm (n_tile -1: IDP4A, lane = row, S K segments, 4 / 8 columns per warp,
    ragged column tiles) equals the oracle's fmaf((float)acc, s, b) and the epilogue's ReLU /
    sigmoid / Q element by element."""
    rng = np.random.default_rng(epi * 1000 + Mr * 7 + K)
    x = rng.normal(0, 1.0, size=(Mr, K)).astype(np.float32)
    W = rng.uniform(-0.08, 0.08, size=(N, K)).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, size=N).astype(np.float32) if bias else None
    qa, qw = O.quantize(x), O.quantize(W)
    v = O.linear(qa, qw, b, CLIP)
    A, Wd = to_dev(qa), to_dev(qw)
    bd = to_dev(b) if bias else None
    of = empty((Mr, N), torch.float32)
    oq = empty((Mr, N), torch.int8)
    bp = ptr(bd) if bias else None
    if epi == M.EPI_RELU_Q:
        M.op_gemm_i8(ptr(A), ptr(Wd), Mr, N, K, bp, CLIP, epi, ptr(oq), None, -1)
    else:
        M.op_gemm_i8(ptr(A), ptr(Wd), Mr, N, K, bp, CLIP, epi, ptr(of), ptr(oq), -1)
    sync()
    r = np.maximum(v, np.float32(0))
    if epi in (M.EPI_F32, M.EPI_F32_Q):
        assert np.array_equal(of.cpu().numpy(), v)
    if epi == M.EPI_F32_Q:
        assert np.array_equal(oq.cpu().numpy(), O.quantize(v))
    if epi == M.EPI_RELU_Q:
        assert np.array_equal(oq.cpu().numpy(), O.quantize(r))
    if epi == M.EPI_RELU_F32_Q:
        assert np.array_equal(of.cpu().numpy(), r)
        assert np.array_equal(oq.cpu().numpy(), O.quantize(r))
    if epi == M.EPI_SIGMOID:
        assert np.array_equal(of.cpu().numpy(), O.sigmoid_array(v))


# swap-AB tcgen05 kernel (n_tile -2: W's 128-row tiles as the MMA's M operand, the M <= 128 rows
# of A as its N = 16 / 32 / 64 / 128 operand; deep K split over a cluster)
SAB_SHAPES = [
    (1, 256, 256, 1), (8, 1024, 1024, 1), (16, 3072, 1024, 1), (17, 1024, 1024, 2),
    (32, 4096, 1024, 1), (33, 1024, 4096, 1), (64, 1024, 4096, 4), (50, 208, 192, 1),
    (100, 512, 2048, 2), (128, 1024, 1024, 8), (5, 36000, 256, 1), (29, 160, 1040, 4),
    (63, 1024, 8192, 1),
]


@pytest.mark.parametrize("Mr,N,K,ks", SAB_SHAPES)
def test_gemm_swap_ab_acc_bitexact(Mr, N, K, ks):
    a = rand_codes((Mr, K), Mr + K + 3)
    w = rand_codes((N, K), N + 11)
    out = empty((Mr, N), torch.int32)
    M.op_gemm_i8_split(ptr(to_dev(a)), ptr(to_dev(w)), Mr, N, K, None, CLIP, M.EPI_ACC, ptr(out), None, -2, ks)
    sync()
    assert np.array_equal(out.cpu().numpy(), O.gemm_acc(a, w))


@pytest.mark.parametrize("epi", [M.EPI_F32, M.EPI_F32_Q, M.EPI_RELU_Q, M.EPI_RELU_F32_Q, M.EPI_SIGMOID])
@pytest.mark.parametrize("Mr,N,K,ks,bias", [(1, 256, 256, 1, True), (12, 1024, 1024, 1, True),
                                            (32, 1024, 4096, 4, True), (47, 2048, 512, 1, False),
                                            (64, 4096, 1024, 2, True), (90, 160, 256, 1, True),
                                            (128, 512, 2048, 1, True)])
def test_gemm_swap_ab_epilogues_bitexact(epi, Mr, N, K, ks, bias):
    """k_gemm_sab equals the oracle's fmaf((float)acc, s, b) and the ReLU / sigmoid / Q epilogue
    element by element (ragged column tiles, split-K clusters, every row-tile width)."""
    rng = np.random.default_rng(epi * 977 + Mr * 3 + K)
    x = rng.normal(0, 1.0, size=(Mr, K)).astype(np.float32)
    W = rng.uniform(-0.08, 0.08, size=(N, K)).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, size=N).astype(np.float32) if bias else None
    qa, qw = O.quantize(x), O.quantize(W)
    v = O.linear(qa, qw, b, CLIP)
    A, Wd = to_dev(qa), to_dev(qw)
    bp = ptr(to_dev(b)) if bias else None
    of = empty((Mr, N), torch.float32)
    oq = empty((Mr, N), torch.int8)
    if epi == M.EPI_RELU_Q:
        M.op_gemm_i8_split(ptr(A), ptr(Wd), Mr, N, K, bp, CLIP, epi, ptr(oq), None, -2, ks)
    else:
        M.op_gemm_i8_split(ptr(A), ptr(Wd), Mr, N, K, bp, CLIP, epi, ptr(of), ptr(oq), -2, ks)
    sync()
    r = np.maximum(v, np.float32(0))
    if epi in (M.EPI_F32, M.EPI_F32_Q):
        assert np.array_equal(of.cpu().numpy(), v)
    if epi == M.EPI_F32_Q:
        assert np.array_equal(oq.cpu().numpy(), O.quantize(v))
    if epi == M.EPI_RELU_Q:
        assert np.array_equal(oq.cpu().numpy(), O.quantize(r))
    if epi == M.EPI_RELU_F32_Q:
        assert np.array_equal(of.cpu().numpy(), r)
        assert np.array_equal(oq.cpu().numpy(), O.quantize(r))
    if epi == M.EPI_SIGMOID:
        assert np.array_equal(of.cpu().numpy(), O.sigmoid_array(v))


@pytest.mark.parametrize("Mr,N,K", [(1, 36000, 1024), (9, 36000, 256), (40, 36000, 512), (128, 50, 32)])
def test_gemm_swap_ab_argmax_bitexact_with_ties(Mr, N, K):
    """The swap-AB argmax epilogue (warp-wide max of packed (v, column) keys per row) picks the
    lowest column among exact ties, as the oracle's first maximum does (R15)."""
    rng = np.random.default_rng(Mr + N + K)
    x = rng.normal(0, 1.0, size=(Mr, K)).astype(np.float32)
    E = rng.uniform(-0.5, 0.5, size=(N, K)).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, size=N).astype(np.float32)
    qa, qE = O.quantize(x), O.quantize(E)
    best = np.argmax(O.linear(qa, qE, b, CLIP), axis=1)
    for i in range(0, Mr, 2):   # exact ties: the winner copied to a lower and a higher column
        j = int(best[i])
        for j2 in ((j * 7 + 11) % N, (j + N // 2) % N, j ^ 1 if (j ^ 1) < N else j):
            if j2 != j:
                qE[j2] = qE[j]
                b[j2] = b[j]
    ref = np.argmax(O.linear(qa, qE, b, CLIP), axis=1)
    keys = zeros((Mr,), torch.int64)
    M.op_gemm_i8(ptr(to_dev(qa)), ptr(to_dev(qE)), Mr, N, K, ptr(to_dev(b)), CLIP, M.EPI_ARGMAX, ptr(keys), None, -2)
    ids = empty((Mr,), torch.int32)
    M.op_argmax_ids(ptr(keys), Mr, ptr(ids))
    sync()
    assert np.array_equal(ids.cpu().numpy(), ref)


# CTA-pair persistent kernel (n_tile -3: 256 x 256 tiles on a 2-CTA cluster, tcgen05 cta_group::2)
PAIR_SHAPES = [(256, 256, 128), (257, 304, 256), (1000, 1024, 1024), (5000, 3072, 1024), (130, 36000, 256),
               (4097, 2048, 1040), (1, 256, 64)]


@pytest.mark.parametrize("Mr,N,K", PAIR_SHAPES)
def test_gemm_pair_acc_bitexact(Mr, N, K):
    a = rand_codes((Mr, K), Mr + K + 5)
    w = rand_codes((N, K), N + 13)
    out = empty((Mr, N), torch.int32)
    M.op_gemm_i8(ptr(to_dev(a)), ptr(to_dev(w)), Mr, N, K, None, CLIP, M.EPI_ACC, ptr(out), None, -3)
    sync()
    assert np.array_equal(out.cpu().numpy(), O.gemm_acc(a, w))


@pytest.mark.parametrize("epi", [M.EPI_F32, M.EPI_F32_Q, M.EPI_RELU_Q, M.EPI_RELU_F32_Q, M.EPI_SIGMOID])
@pytest.mark.parametrize("Mr,N,K", [(600, 1024, 1024), (3001, 4096, 256), (77, 160, 512)])
def test_gemm_pair_epilogues_bitexact(epi, Mr, N, K):
    rng = np.random.default_rng(epi * 31 + Mr)
    x = rng.normal(0, 1.0, size=(Mr, K)).astype(np.float32)
    W = rng.uniform(-0.08, 0.08, size=(N, K)).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, size=N).astype(np.float32)
    qa, qw = O.quantize(x), O.quantize(W)
    v = O.linear(qa, qw, b, CLIP)
    A, Wd, bd = to_dev(qa), to_dev(qw), to_dev(b)
    of = empty((Mr, N), torch.float32)
    oq = empty((Mr, N), torch.int8)
    if epi == M.EPI_RELU_Q:
        M.op_gemm_i8(ptr(A), ptr(Wd), Mr, N, K, ptr(bd), CLIP, epi, ptr(oq), None, -3)
    else:
        M.op_gemm_i8(ptr(A), ptr(Wd), Mr, N, K, ptr(bd), CLIP, epi, ptr(of), ptr(oq), -3)
    sync()
    r = np.maximum(v, np.float32(0))
    if epi in (M.EPI_F32, M.EPI_F32_Q):
        assert np.array_equal(of.cpu().numpy(), v)
    if epi == M.EPI_F32_Q:
        assert np.array_equal(oq.cpu().numpy(), O.quantize(v))
    if epi == M.EPI_RELU_Q:
        assert np.array_equal(oq.cpu().numpy(), O.quantize(r))
    if epi == M.EPI_RELU_F32_Q:
        assert np.array_equal(of.cpu().numpy(), r)
        assert np.array_equal(oq.cpu().numpy(), O.quantize(r))
    if epi == M.EPI_SIGMOID:
        assert np.array_equal(of.cpu().numpy(), O.sigmoid_array(v))


@pytest.mark.parametrize("Mr,K", [(630, 1024), (3000, 256)])
def test_gemm_pair_argmax_bitexact_with_ties(Mr, K):
    N = 36000
    rng = np.random.default_rng(Mr + K + 7)
    x = rng.normal(0, 1.0, size=(Mr, K)).astype(np.float32)
    E = rng.uniform(-0.5, 0.5, size=(N, K)).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, size=N).astype(np.float32)
    qa, qE = O.quantize(x), O.quantize(E)
    best = np.argmax(O.linear(qa, qE, b, CLIP), axis=1)
    for i in range(0, Mr, 5):
        j = int(best[i])
        for j2 in ((j * 7 + 11) % N, (j + N // 2) % N):
            if j2 != j:
                qE[j2] = qE[j]
                b[j2] = b[j]
    ref = np.argmax(O.linear(qa, qE, b, CLIP), axis=1)
    keys = zeros((Mr,), torch.int64)
    M.op_gemm_i8(ptr(to_dev(qa)), ptr(to_dev(qE)), Mr, N, K, ptr(to_dev(b)), CLIP, M.EPI_ARGMAX, ptr(keys), None, -3)
    ids = empty((Mr,), torch.int32)
    M.op_argmax_ids(ptr(keys), Mr, ptr(ids))
    sync()
    assert np.array_equal(ids.cpu().numpy(), ref)


def test_gemm_swap_ab_rejects():
    """n_tile -2 is an argument error (never a silent fallback) beyond 128 rows."""
    a = to_dev(rand_codes((129, 64), 1))
    w = to_dev(rand_codes((64, 64), 2))
    out = empty((129, 64), torch.int32)
    with pytest.raises(Exception):
        M.op_gemm_i8(ptr(a), ptr(w), 129, 64, 64, None, CLIP, M.EPI_ACC, ptr(out), None, -2)


@pytest.mark.parametrize("Mr,N,K,bias", [(3, 50, 32, True), (200, 36000, 256, True),
                                         (129, 36000, 192, False), (390, 36000, 512, True),
                                         (650, 36000, 256, True)])   # persistent kernel
def test_gemm_argmax_bitexact_with_ties(Mr, N, K, bias):
    rng = np.random.default_rng(Mr + N)
    x = rng.normal(0, 1.0, size=(Mr, K)).astype(np.float32)
    E = rng.uniform(-0.5, 0.5, size=(N, K)).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, size=N).astype(np.float32) if bias else None
    qa, qE = O.quantize(x), O.quantize(E)
    logits = O.linear(qa, qE, b, CLIP)
    best = np.argmax(logits, axis=1)
    # exact ties: copy each row's winner (code row and bias) to a LOWER and a HIGHER column
    for i in range(0, Mr, 3):
        j = int(best[i])
        for j2 in ((j * 7 + 11) % N, (j + N // 2) % N):
            if j2 != j:
                qE[j2] = qE[j]
                if b is not None:
                    b[j2] = b[j]
    logits = O.linear(qa, qE, b, CLIP)
    ref = np.argmax(logits, axis=1)                   # first maximum = lowest id (R15)
    keys = zeros((Mr,), torch.int64)
    M.op_gemm_i8(ptr(to_dev(qa)), ptr(to_dev(qE)), Mr, N, K, ptr(to_dev(b)) if b is not None else None,
                 CLIP, M.EPI_ARGMAX, ptr(keys))
    ids = empty((Mr,), torch.int32)
    M.op_argmax_ids(ptr(keys), Mr, ptr(ids))
    sync()
    assert np.array_equal(ids.cpu().numpy(), ref)


# ------------------------------------------------------------------ LayerNorm (+gate) (A6-A8)
@pytest.mark.parametrize("d", [192, 256, 512, 1024])
@pytest.mark.parametrize("gate", [False, True])
def test_layernorm(d, gate):
    n = 333
    x, dl = synth.uniform_activations((n, d), 1, 2.0), synth.uniform_activations((n, d), 2, 2.0)
    g = synth.uniform_activations((d,), 3, 0.1) + np.float32(1)
    b = synth.uniform_activations((d,), 4, 0.1)
    gi = synth.uniform_activations((n, d), 5, 3.0) if gate else None     # gate logits
    gf = synth.uniform_activations((n, d), 6, 3.0) if gate else None
    ref = O.residual_ln(x, dl, g, b, 1e-6, O.sigmoid_array(gi) if gate else None,
                        O.sigmoid_array(gf) if gate else None)
    out = empty((n, d), torch.float32)
    oq = empty((n, d), torch.int8)
    M.op_layernorm(ptr(to_dev(x)), ptr(to_dev(dl)), ptr(to_dev(gi)) if gate else None,
                   ptr(to_dev(gf)) if gate else None, ptr(to_dev(g)), ptr(to_dev(b)), n, d, 1e-6,
                   CLIP, ptr(out), ptr(oq))
    sync()
    got = out.cpu().numpy()
    assert np.mean(got == ref) > 0.9999
    np.testing.assert_allclose(got, ref, rtol=1e-6, atol=1e-6)
    assert not boundary_explained(ref, O.quantize(ref), oq.cpu().numpy()).any()


# ------------------------------------------------------------------ AAN running sum (A6)
def test_aan_step_bitexact():
    n, d, T = 70, 256, 9
    Y = synth.uniform_activations((T, n, d), 8, 3.0)
    Cd = zeros((n, d), torch.float32)
    g = empty((n, d), torch.float32)
    gq = empty((n, d), torch.int8)
    ref_G = np.stack([O.aan_average(Y[:, i, :]) for i in range(n)], axis=1)   # [T, n, d]
    for t in range(T):
        M.op_aan_step(ptr(Cd), ptr(to_dev(Y[t])), n, d, t + 1, CLIP, ptr(g), ptr(gq))
        sync()
        assert np.array_equal(g.cpu().numpy(), ref_G[t])
        assert np.array_equal(gq.cpu().numpy(), O.quantize(ref_G[t]))


# ------------------------------------------------------------------ embedding (A2, A5)
@pytest.mark.parametrize("d", [192, 512])
def test_embed_bitexact(d):
    V = 1000
    E = synth.uniform_activations((V, d), 9, 0.5)
    rng = np.random.default_rng(d)
    ids = rng.integers(-1, V, size=300).astype(np.int32)
    pos = rng.integers(0, 512, size=300).astype(np.int32)
    x = empty((300, d), torch.float32)
    xq = empty((300, d), torch.int8)
    M.op_embed(ptr(to_dev(E)), d, ptr(to_dev(ids)), ptr(to_dev(pos)), 300, CLIP, ptr(x), ptr(xq))
    sync()
    ref = O.embed_rows(E, ids, pos)
    assert np.array_equal(x.cpu().numpy(), ref)
    assert np.array_equal(xq.cpu().numpy(), O.quantize(ref))


# ------------------------------------------------------------------ attention (A3, A7)
@pytest.mark.parametrize("d,H", [(192, 8), (256, 8), (512, 8), (1024, 16)])
def test_attention(d, H):
    rng = np.random.default_rng(d + H)
    lens = rng.integers(0, 101, size=40).astype(np.int32)
    lens[0], lens[1] = 1, 100
    starts = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int32)
    S = int(lens.sum())
    kv = rng.normal(0, 1, size=(S, 2 * d)).astype(np.float32)        # K | V per row
    q = rng.normal(0, 1, size=(40, d)).astype(np.float32)
    oq = empty((40, d), torch.int8)
    of = empty((40, d), torch.float32)
    M.op_attention(ptr(to_dev(q)), d, ptr(to_dev(kv)), 2 * d, 0, d, ptr(to_dev(starts)),
                   ptr(to_dev(lens)), 40, d, H, CLIP, ptr(oq), ptr(of))
    sync()
    ref = np.zeros((40, d), np.float32)
    for r in range(40):
        if lens[r] > 0:
            blk = kv[starts[r]:starts[r] + lens[r]]
            ref[r] = O.attention(q[r], blk[:, :d], blk[:, d:], H)
    got = of.cpu().numpy()
    assert np.mean(got == ref) > 0.9999
    np.testing.assert_allclose(got, ref, rtol=1e-6, atol=1e-7)
    assert not boundary_explained(ref, O.quantize(ref), oq.cpu().numpy()).any()


@pytest.mark.parametrize("d,H,smax", [(256, 4, 100), (1024, 16, 40), (512, 8, 97), (1024, 16, 7)])
def test_attention_enc_variants(d, H, smax):
    """mnmt_op_attention_enc: the d_h = 64 multi-query encoder kernel (4 / 8 queries per warp pass,
    sentences of 1..smax tokens, ragged last passes) writes exactly the generic warp-per-query
    kernel's codes, and both are the oracle's Q(attention) up to boundary-explained flips."""
    rng = np.random.default_rng(d + smax)
    n_sent = 37
    lens = rng.integers(1, smax + 1, size=n_sent).astype(np.int32)
    lens[0], lens[-1] = 1, smax
    starts = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int32)
    rows = int(lens.sum())
    qkv = rng.normal(0, 1, size=(rows, 3 * d)).astype(np.float32)
    qd, sd, ld = to_dev(qkv), to_dev(starts), to_dev(lens)
    outs = []
    for variant in (1, 2, 3, 0):
        oq = zeros((rows, d), torch.int8)
        M.op_attention_enc(ptr(qd), ptr(sd), ptr(ld), n_sent, d, H, smax, CLIP, ptr(oq), variant)
        sync()
        outs.append(oq.cpu().numpy())
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
    ref = np.zeros((rows, d), np.float32)
    for s in range(n_sent):
        blk = qkv[starts[s]:starts[s] + lens[s]]
        for i in range(lens[s]):
            ref[starts[s] + i] = O.attention(blk[i, :d], blk[:, d:2 * d], blk[:, 2 * d:], H)
    rq = O.quantize(ref)
    assert not boundary_explained(ref, rq, outs[0]).any()
    assert np.mean(outs[0] != rq) < 1e-4


@pytest.mark.parametrize("d,H", [(256, 8), (512, 8), (1024, 16), (192, 8)])
def test_src_attention_tma(d, H):
    """mnmt_op_src_attention (the decode path's choice: TMA-tiled K / V for d/H = 32 / 64,
    spans of 0..130 crossing several 32-position chunks, rows at the end of the K/V buffer) equals
    the oracle's attention and the generic kernel's output bit for bit."""
    rng = np.random.default_rng(d + H + 5)
    n = 50
    lens = rng.integers(0, 131, size=n).astype(np.int32)
    lens[0], lens[1], lens[2], lens[-1] = 1, 130, 0, 33
    starts = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int32)
    S = int(lens.sum())
    kv = rng.normal(0, 1, size=(S, 2 * d)).astype(np.float32)
    q = rng.normal(0, 1, size=(n, d)).astype(np.float32)
    oq, of = empty((n, d), torch.int8), empty((n, d), torch.float32)
    oq2, of2 = empty((n, d), torch.int8), empty((n, d), torch.float32)
    kd, qd, sd, ld = to_dev(kv), to_dev(q), to_dev(starts), to_dev(lens)
    M.op_src_attention(ptr(qd), d, ptr(kd), S, 2 * d, 0, d, ptr(sd), ptr(ld), int(lens.max()), n, d, H,
                       CLIP, ptr(oq), ptr(of))
    M.op_attention(ptr(qd), d, ptr(kd), 2 * d, 0, d, ptr(sd), ptr(ld), n, d, H, CLIP, ptr(oq2), ptr(of2))
    sync()
    got = of.cpu().numpy()
    assert np.array_equal(got, of2.cpu().numpy())
    assert np.array_equal(oq.cpu().numpy(), oq2.cpu().numpy())
    ref = np.zeros((n, d), np.float32)
    for r in range(n):
        if lens[r] > 0:
            blk = kv[starts[r]:starts[r] + lens[r]]
            ref[r] = O.attention(q[r], blk[:, :d], blk[:, d:], H)
    assert np.mean(got == ref) > 0.9999
    np.testing.assert_allclose(got, ref, rtol=1e-6, atol=1e-7)
    assert not boundary_explained(ref, O.quantize(ref), oq.cpu().numpy()).any()


@pytest.mark.parametrize("d,H,n", [(1024, 16, 630), (512, 8, 300), (256, 4, 200)])
def test_src_attention_f32_option(d, H, n):
    """The fp32 variant of the one-warp TMA attention (option attn_f32): context within 4e-6 of the
    fp64 oracle relative to the row's scale, every code equal to the oracle's or a boundary-explained
    flip (x * sigma within 1e-4 relative of a rounding midpoint), and the flips rare."""
    rng = np.random.default_rng(d + n + 3)
    lens = rng.integers(1, 60, size=n).astype(np.int32)
    starts = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int32)
    S = int(lens.sum())
    kv = rng.normal(0, 1, size=(S, 2 * d)).astype(np.float32)
    q = rng.normal(0, 1, size=(n, d)).astype(np.float32)
    oq, of = zeros((n, d), torch.int8), zeros((n, d), torch.float32)
    M.op_src_attention_f32(ptr(to_dev(q)), d, ptr(to_dev(kv)), S, 2 * d, 0, d, ptr(to_dev(starts)), ptr(to_dev(lens)),
                           int(lens.max()), n, d, H, CLIP, ptr(oq), ptr(of))
    sync()
    ref = np.zeros((n, d), np.float32)
    for r in range(n):
        blk = kv[starts[r]:starts[r] + lens[r]]
        ref[r] = O.attention(q[r], blk[:, :d], blk[:, d:], H)
    got = of.cpu().numpy()
    scale = np.maximum(np.abs(ref), np.sqrt(np.mean(ref.astype(np.float64) ** 2, axis=1, keepdims=True)))
    assert np.max(np.abs(got - ref) / scale) < 4e-6
    rq, gq = O.quantize(ref), oq.cpu().numpy()
    assert not boundary_explained(ref, rq, gq, rel=1e-4).any()
    assert np.mean(gq != rq) < 1e-3


# ------------------------------------------------------------------ A11 across GPUs (unshard)
def test_gather_rows():
    """mnmt_op_gather_rows puts the all-gathered rows of a strong-scaling job back in input order:
    the same result as the plan's numpy twin (paper_1805_12096_b200.dist.unshard_host)."""
    from paper_1805_12096_b200 import dist as D
    rng = np.random.default_rng(4)
    n, world = 300, 4
    ml = rng.integers(0, 30, size=n)
    outs = [rng.integers(3, 36000, size=rng.integers(0, m + 1)).astype(np.int32) for m in ml]
    lengths = rng.integers(1, 50, size=n)
    shards = [D.shard_round_robin(lengths, r, world) for r in range(world)]
    plan = D.gather_plan(ml, shards)
    gi = np.zeros(plan.world * plan.id_cap, np.int32)
    gl = np.zeros(plan.world * plan.n_cap, np.int32)
    for r, s in enumerate(shards):
        f, l = D.pack_ids([outs[i] for i in s], ml[s])
        gi[r * plan.id_cap:r * plan.id_cap + len(f)] = f
        gl[r * plan.n_cap:r * plan.n_cap + len(l)] = l
    un = D.DeviceUnshard(plan, torch_dev())
    ids, ln = un(to_dev(gi), to_dev(gl))
    sync()
    ref_ids, ref_ln = D.unshard_host(gi, gl, plan)
    ln_h = ln.cpu().numpy()
    assert np.array_equal(ln_h, ref_ln)
    got = D.split_rows(ids.cpu().numpy(), ln_h, ml)
    assert all(np.array_equal(a, b) for a, b in zip(got, outs))
