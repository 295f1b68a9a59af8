"""Element-wise tolerances for comparing GPU weight gradients with the oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): a tolerance computed from the oracle's own
recorded activations; nothing here is part of the method.

The GPU rounds both operands of every dense product to TF32 (reading R2) and accumulates in
FP32; the oracle run with ``operand_rounding="tf32"`` and the GPU's layer ``orders`` (reading Q7)
rounds the same operands and accumulates exactly.  What separates the two:

1. accumulation order inside each weight-gradient product dW_l = A_lᵀ·B_l, bounded by the north
   star's GEMM tolerance applied to that product: ``gemm_rtol·|A_l|ᵀ·|B_l|`` (SURVEY c.5 "the
   GEMM bound");
2. ReLU-mask decisions (reading Q8, ReLU'(0) := 0) that FP32 accumulation can flip: where
   ``|Z_l| <= eps_acc·Zmag_l`` (Zmag = the magnitude product of Z_l's own GEMM and aggregation)
   either mask value is a correct rounding of the same Z_l.  A flipped mask moves dZ_l by the
   whole |dH_l| there (not a relative error), and H_l by at most ``eps_acc·Zmag_l``; both reach
   dW through the same products and are carried down the backward pass as magnitudes.

``eps_acc`` (1e-4 by default, ~840 FP32 ulps) covers the FP32 accumulation of the forward GEMM
(K <= 602 terms) and of the aggregation (hub rows in blocks of 256 edges).  The bound is first
order in these errors.  It does not cover the rarer decision the two sides can take differently
when a stored operand straddles a TF32 rounding boundary (one TF32 ulp, 2^-10 relative, apart)
next to a near-zero pre-activation; where that lands in an otherwise fully masked (near-dead)
unit the bound is ~0 while the flipped term is not, so the tests add an absolute floor of 1e-5 of
the matrix's largest |dW*| (``FLOOR_REL``), far below the north star's 2e-3.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .gcn_oracle import a_hat_values, csr_matmul

__all__ = ["tf32_gradient_bounds", "FLOOR_REL"]

FLOOR_REL = 1e-5


def tf32_gradient_bounds(g, cache, Ws, bs, agg: str = "gcn", gemm_rtol: float = 2e-3, eps_acc: float = 1e-4,
                         release: bool = False, dtype=np.float64):
    """(bW, bb): element-wise bounds on |dW_l − dW*_l| and |db_l − db*_l| between the GPU and the
    oracle run with operand_rounding="tf32" and the same orders (module docstring).  ``cache`` is
    that oracle's forward/backward cache (H, Z, Y, dZ, dH, orders).  release=True drops the
    cache's per-layer arrays as they are used (full-size workloads); dtype sets the precision of
    the magnitude products (FP32 suffices for a tolerance)."""
    L = len(Ws)
    orders = cache["orders"]
    # the aggregation as a CSR in the bound's dtype (full-size FP32 magnitudes stay FP32)
    vals = a_hat_values(g) if agg == "gcn" else np.ones(g.nnz)
    A_csr = sp.csr_matrix((vals.astype(dtype), g.col_idx, g.row_ptr), shape=(g.num_nodes, g.num_nodes))
    dcol = g.deg.astype(dtype)[:, None]

    def AGG(M, tr=False):   # gcn Â (= Âᵀ), sum Ã (= Ãᵀ), mean D̃⁻¹Ã / Ã·D̃⁻¹ (aggregate_scheme's definitions)
        if agg not in ("gcn", "sum", "mean"):
            raise ValueError(agg)
        M = np.asarray(M, dtype=dtype)
        if agg == "mean":
            return csr_matmul(A_csr, M / dcol) if tr else csr_matmul(A_csr, M) / dcol
        return csr_matmul(A_csr, M)

    Wa = [np.abs(np.asarray(W, dtype=dtype)) for W in Ws]
    ba = [np.abs(np.asarray(b, dtype=dtype)) for b in bs]
    def mag(a):   # |a| in dtype, in row chunks (no full-size FP64 temporary)
        if sp.issparse(a):
            return np.abs(a.toarray()).astype(dtype, copy=False)
        a = np.asarray(a)
        out = np.empty(a.shape, dtype=dtype)
        step = max(1, (1 << 24) // max(1, a.shape[-1] if a.ndim > 1 else 1))
        for i in range(0, a.shape[0], step):
            out[i:i + step] = np.abs(a[i:i + step])
        return out

    def where_amb(m, a):   # a (as |a| in dtype) where m, else 0, in row chunks
        a = np.asarray(a)
        out = np.zeros(a.shape, dtype=dtype)
        step = max(1, (1 << 24) // max(1, a.shape[1]))
        for i in range(0, a.shape[0], step):
            np.copyto(out[i:i + step], np.abs(a[i:i + step]), where=m[i:i + step], casting="unsafe")
        return out

    # forward: the ambiguous ReLU decisions of every hidden layer, and eps_acc·Zmag there
    amb, hflip = [None] * L, [None] * L
    for l in range(L - 1):
        if orders[l] == "AF":
            zmag = mag(cache["Y"][l]) @ Wa[l]
        else:
            zmag = AGG(mag(cache["H"][l]) @ Wa[l])
        zmag += ba[l]
        zmag *= eps_acc
        Z = cache["Z"][l]
        amb[l] = np.empty(zmag.shape, dtype=bool)
        step = max(1, (1 << 24) // zmag.shape[1])
        for i in range(0, zmag.shape[0], step):
            amb[l][i:i + step] = np.abs(Z[i:i + step]) <= zmag[i:i + step]
        hflip[l] = sp.csr_matrix(where_amb(amb[l], zmag))   # eps_acc·Zmag, nonzero on amb only
        del zmag

    bW, bb = [None] * L, [None] * L
    F = None   # flip-induced error magnitude of dZ_l (unscaled), None = 0
    for l in range(L - 1, -1, -1):
        dZa = mag(cache["dZ"][l])
        if orders[l] == "AF":
            A = mag(cache["Y"][l])
            Bm = dZa
            Bf = F
            A_flip = None   # Y = AGG(H_{l-1}); a flipped H feeds it through AGG
            if l > 0 and hflip[l - 1] is not None:
                A_flip = AGG(hflip[l - 1].toarray())
        else:
            A = mag(cache["H"][l])
            Bm = AGG(dZa, True)
            Bf = AGG(F, True) if F is not None else None
            A_flip = hflip[l - 1] if l > 0 else None
        b = gemm_rtol * (A.T @ Bm)
        if Bf is not None:
            b += A.T @ Bf
        if A_flip is not None:
            b += np.asarray(A_flip.T @ (Bm if Bf is None else Bm + Bf))
        bW[l] = b.astype(np.float64)
        bb[l] = gemm_rtol * dZa.sum(axis=0, dtype=np.float64)
        if F is not None:
            bb[l] += F.sum(axis=0, dtype=np.float64)
        if l > 0:
            # dH_{l-1} = B·W_lᵀ (TF: G_l·W_lᵀ; AF: AGGᵀ(dZ_l·W_lᵀ)): the flip error of B rides along,
            # and layer l-1's own ambiguous decisions add the whole |dH_{l-1}|
            if Bf is None:
                Fh = None
            elif orders[l] == "AF":
                Fh = AGG(Bf @ Wa[l].T, True)
            else:
                Fh = Bf @ Wa[l].T
            mask = np.asarray(cache["Z"][l - 1]) > 0.0
            Fn = where_amb(amb[l - 1], cache["dH"][l - 1])
            if Fh is not None:
                Fn += np.where(mask | amb[l - 1], Fh, 0.0)
            F = Fn
        del A, Bm, Bf, dZa
        if release:
            cache["dZ"][l] = cache["dH"][l] = None
            if cache["Y"] and l < len(cache["Y"]):
                cache["Y"][l] = None
            if l + 1 < len(cache["H"]):
                cache["H"][l + 1] = None
            cache["Z"][l] = None
    return bW, bb
