"""Shared helpers for the -m gpu parity tests (inputs from synth/, references from oracle/)."""
from __future__ import annotations

import numpy as np
import torch

import oracle


def cuda(a, dtype=None):
    t = torch.as_tensor(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def padded(x: np.ndarray, width: int) -> np.ndarray:
    out = np.zeros((x.shape[0], width), dtype=x.dtype)
    out[:, :x.shape[1]] = x
    return out


def pad_width(w: int) -> int:
    return 4 if w <= 4 else (w + 7) // 8 * 8


def agg_bound(g: "oracle.Graph", T: np.ndarray) -> np.ndarray:
    """(|Â|·|T|) — the magnitude sum the FP32 aggregation tolerance is relative to (SURVEY c.5)."""
    return oracle.aggregate(g, np.abs(T.astype(np.float64)))


def assert_agg_close(Z, Zref, bound, rtol=1e-5, extra=0.0, what="aggregation"):
    Z = np.asarray(Z, np.float64)
    err = np.abs(Z - Zref)
    lim = rtol * (bound + extra) + 1e-30
    ratio = float((err / lim).max()) if err.size else 0.0
    assert ratio <= 1.0, f"{what}: max |err| / (rtol*bound) = {ratio:.3g}"
    return ratio


def assert_gemm_close(C, A, B, Cref=None, rtol=2e-3, what="gemm"):
    """|C - C*| <= 2e-3 (|A|·|B|) elementwise (SURVEY c.5, TF32 operands)."""
    A64, B64 = np.asarray(A, np.float64), np.asarray(B, np.float64)
    ref = A64 @ B64 if Cref is None else Cref
    bound = np.abs(A64) @ np.abs(B64)
    err = np.abs(np.asarray(C, np.float64) - ref)
    ratio = float((err / (rtol * bound + 1e-30)).max()) if err.size else 0.0
    assert ratio <= 1.0, f"{what}: max |err| / (2e-3 |A||B|) = {ratio:.3g}"
    return ratio
