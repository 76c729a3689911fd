"""Helpers for the -m gpu parity tests (device memory through torch; kernels through the C-ABI)."""
import numpy as np

import oracle.oracle as O


def torch_dev():
    import torch
    return torch.device("cuda:0")


_KEEP = []   # device temporaries stay alive until the test ends (raw pointers go to the C-ABI)


def release():
    _KEEP.clear()


def to_dev(a):
    import torch
    if a is None:
        return None
    t = torch.from_numpy(np.ascontiguousarray(a)).to(torch_dev())
    _KEEP.append(t)
    return t


def empty(shape, dtype):
    import torch
    return torch.empty(shape, dtype=dtype, device=torch_dev())


def zeros(shape, dtype):
    import torch
    return torch.zeros(shape, dtype=dtype, device=torch_dev())


def ptr(t):
    return None if t is None else t.data_ptr()


def sync():
    import torch
    torch.cuda.synchronize()


def boundary_explained(x_ref: np.ndarray, q_ref: np.ndarray, q_got: np.ndarray, x_got=None,
                       rel: float = 1e-5, clip: float = 2.0) -> np.ndarray:
    """P-2 'boundary-explained' code flips: a code may differ from the oracle's only if the
    oracle's x*sigma lies within the float drift of a rounding midpoint k+1/2 (|dq| == 1).
    Returns a bool mask of UNEXPLAINED mismatches."""
    mism = q_ref != q_got
    if not mism.any():
        return mism
    sig = np.float32(127.0) / np.float32(clip)
    v = np.clip(x_ref.astype(np.float64), -clip, clip) * float(sig)
    frac = np.abs(v - np.floor(v) - 0.5)
    tol = rel * np.maximum(np.abs(v), 1.0)
    ok = (np.abs(q_ref.astype(np.int32) - q_got.astype(np.int32)) == 1) & (frac <= tol)
    return mism & ~ok


def near_tie_allowance(flipped_dq: np.ndarray, qE: np.ndarray, s: float) -> float:
    """Top-2 margin under which a differing argmax is explainable by code flips of the final
    layer output: 2*s*sum|dq_k|*max_j|qE[j,k]|."""
    if not flipped_dq.any():
        return 0.0
    return 2.0 * s * float(np.sum(np.abs(flipped_dq) * np.abs(qE).max(axis=0)))


def check_forced_steps(gpu_ids, gpu_codes, trace, qE, s):
    """Per-step token ids must be bit-exact except near-ties explained by output-code flips.
    Returns (n_steps, n_exact, n_flagged)."""
    n = len(gpu_ids)
    exact = int(np.sum(gpu_ids == trace["ids"]))
    flagged = 0
    for t in np.nonzero(gpu_ids != trace["ids"])[0]:
        dq = gpu_codes[t].astype(np.int32) - trace["out_codes"][t].astype(np.int32)
        allow = near_tie_allowance(dq, qE, s)
        assert trace["margin"][t] <= allow + 1e-6, (
            f"step {t}: gpu id {gpu_ids[t]} vs oracle {trace['ids'][t]}, margin "
            f"{trace['margin'][t]} not explained (allowance {allow})")
        flagged += 1
    return n, exact, flagged
