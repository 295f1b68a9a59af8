"""Pins of oracle.bounds.tf32_gradient_bounds (the element-wise gradient tolerance the GPU tests
use against the TF32-operand oracle): an independent FP32 emulation of the GPU's arithmetic —
TF32-rounded GEMM operands, FP32 accumulation, FP32 aggregation, the kernel's layer orders — stays
inside the bound, the bound is tight (a 1 % error of one layer's upstream gradient leaves it), and
it is not vacuous (its median is under 5 % of |dW|).  The bound is used with the absolute floor
oracle.FLOOR_REL·max|dW*| (oracle/bounds.py), as in the GPU tests."""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle
from synth.generate import make_small

pytestmark = pytest.mark.filterwarnings("ignore::RuntimeWarning")


def _emulate_fp32(g, X, Ws, bs, y, agg, orders, dz_scale=1.0):
    """The GPU's arithmetic in numpy FP32: Z = AGG(tf32(H)·tf32(W)) + b (TF) or tf32(AGG(H))·tf32(W)
    + b (AF), ReLU, softmax-CE, backward with the same operand rounding; AGG as an FP32 CSR."""
    n = g.num_nodes
    t32 = lambda a: oracle.tf32_rna(np.asarray(a, np.float32)).astype(np.float32)  # noqa: E731
    if agg == "gcn":
        vals = oracle.a_hat_values(g).astype(np.float32)
    else:
        vals = np.ones(g.nnz, np.float32)
    A = sp.csr_matrix((vals, g.col_idx, g.row_ptr), shape=(n, n))
    L = len(Ws)
    W32 = [np.asarray(W, np.float32) for W in Ws]
    b32 = [np.asarray(b, np.float32) for b in bs]
    H, Z, Y = [np.asarray(X, np.float32)], [], []
    for l in range(L):
        if orders[l] == "AF":
            Y.append(t32(A @ H[l]))
            z = Y[l] @ t32(W32[l]) + b32[l]
        else:
            Y.append(None)
            z = (A @ (t32(H[l]) @ t32(W32[l]))) + b32[l]
        Z.append(z.astype(np.float32))
        if l < L - 1:
            H.append(np.maximum(Z[l], 0))
    z = Z[-1].astype(np.float64)
    p = np.exp(z - z.max(1, keepdims=True))
    p /= p.sum(1, keepdims=True)
    p[np.arange(n), y] -= 1.0
    dZ = (p / n).astype(np.float32) * np.float32(dz_scale)
    dW = [None] * L
    for l in range(L - 1, -1, -1):
        if orders[l] == "AF":
            dW[l] = Y[l].T @ t32(dZ)
            dH = (A.T @ (t32(dZ) @ t32(W32[l]).T)) if l > 0 else None
        else:
            G = A.T @ dZ
            dW[l] = t32(H[l]).T @ t32(G)
            dH = t32(G) @ t32(W32[l]).T if l > 0 else None
        if l > 0:
            dZ = (dH * (Z[l - 1] > 0)).astype(np.float32)
    return dW


@pytest.mark.parametrize("agg,dims,orders", [("gcn", (24, 40, 32, 5), ("AF", "TF", "TF")),
                                             ("gcn", (48, 16, 5), ("TF", "TF")),
                                             ("sum", (24, 32, 16, 5), ("AF", "TF", "TF"))])
def test_fp32_emulation_inside_bound_and_bound_tight(agg, dims, orders):
    w = make_small(1500, 12000, dims[0], dims[-1], seed=21)
    if agg == "sum":
        w["X"] = w["X"] * np.float32(0.125)
    g = oracle.graph_build(w["src"], w["dst"], 1500)
    Ws, bs = oracle.xavier_init(dims, 7)
    bs = [np.asarray(b, np.float32) + np.float32(0.01) for b in bs]
    Z, c = oracle.forward(g, w["X"], Ws, bs, aggregator=agg, operand_rounding="tf32", orders=orders)
    _, dZ = oracle.softmax_ce(Z, w["y"])
    dWt, _ = oracle.backward(g, c, Ws, dZ)
    bW, _ = oracle.tf32_gradient_bounds(g, c, Ws, bs, agg=agg)
    got = _emulate_fp32(g, w["X"], Ws, bs, w["y"], agg, orders)
    for l in range(len(Ws)):
        err = np.abs(got[l].astype(np.float64) - dWt[l])
        bnd = bW[l] + oracle.FLOOR_REL * np.abs(dWt[l]).max()
        assert np.all(err <= bnd), (l, float((err / bnd).max()))
        # not vacuous: the bound is a small fraction of the gradient it guards
        big = np.abs(dWt[l]) > 1e-3 * np.abs(dWt[l]).max()
        assert np.median(bnd[big] / np.abs(dWt[l][big])) < 0.05, l
    # tight: a 1 % error of the output layer's gradient leaves the bound somewhere in every layer
    bad = _emulate_fp32(g, w["X"], Ws, bs, w["y"], agg, orders, dz_scale=1.01)
    for l in range(len(Ws)):
        assert np.any(np.abs(bad[l].astype(np.float64) - dWt[l]) > bW[l] + oracle.FLOOR_REL * np.abs(dWt[l]).max()), l
