"""Pins for the oracle's graph build (G1-G6), Â and aggregation, and the switch (S1-S3).

Every expected value here is derived independently of oracle/: hand cases,
closed forms of Â on named graphs, brute-force re-derivations, and the
paper's printed constants (tests/golden/paper_constants.json).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from synth.generate import make_small

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _naive_csr(src, dst, n):
    """Independent builder: python set per row (SURVEY c.4 'naive std::set-per-row')."""
    rows = [set([u]) for u in range(n)]
    for a, b in zip(src, dst):
        if a != b:
            rows[a].add(b)
            rows[b].add(a)
    ptr = [0]
    cols = []
    for r in rows:
        cols.extend(sorted(r))
        ptr.append(len(cols))
    return np.array(ptr, np.int64), np.array(cols, np.int32)


def _dense_a_hat(src, dst, n):
    """Â from its definition D̃^{-1/2}(A+I)D̃^{-1/2}, built densely (Q1)."""
    A = np.zeros((n, n))
    for a, b in zip(src, dst):
        if a != b:
            A[a, b] = 1.0
            A[b, a] = 1.0
    At = A + np.eye(n)
    d = At.sum(axis=1)
    Dm = np.diag(1.0 / np.sqrt(d))
    return Dm @ At @ Dm


# ---------------------------------------------------------------- G1-G5
def test_hand_case_two_nodes():
    g = oracle.graph_build([0, 1], [1, 0], 2)
    assert g.row_ptr.tolist() == [0, 2, 4]
    assert g.col_idx.tolist() == [0, 1, 0, 1]
    assert g.deg.tolist() == [2, 2]


def test_hand_case_self_loop_and_duplicates():
    # input self loop on 2 is dropped then I added once; duplicate (0,1) collapses
    g = oracle.graph_build([0, 0, 1, 2, 2], [1, 1, 0, 2, 0], 4)
    assert g.row_ptr.tolist() == [0, 3, 5, 7, 8]
    assert g.col_idx.tolist() == [0, 1, 2, 0, 1, 0, 2, 3]
    assert g.deg.tolist() == [3, 2, 2, 1]


def test_errors():
    with pytest.raises(oracle.OracleError) as e:
        oracle.graph_build([0], [3], 3)
    assert e.value.code == "ERANGE"
    with pytest.raises(oracle.OracleError) as e:
        oracle.graph_build([], [], 0)
    assert e.value.code == "EDEGENERATE"


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_against_naive_builder(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 60))
    m = int(rng.integers(0, 200))
    src = rng.integers(0, n, m)
    dst = rng.integers(0, n, m)
    g = oracle.graph_build(src, dst, n)
    ptr, cols = _naive_csr(src.tolist(), dst.tolist(), n)
    assert np.array_equal(g.row_ptr, ptr)
    assert np.array_equal(g.col_idx, cols)
    assert np.array_equal(g.deg, np.diff(ptr).astype(np.int32))


def test_invariants_on_synthetic():
    w = make_small(500, 4000, 8, 3, seed=5)
    g = oracle.graph_build(w["src"], w["dst"], 500)
    assert g.row_ptr[0] == 0 and np.all(np.diff(g.row_ptr) >= 1)
    assert g.row_ptr[-1] == g.nnz == 4000 + 500
    rows = g.rows
    keys = set(zip(rows.tolist(), g.col_idx.tolist()))
    assert all((b, a) in keys for a, b in keys)                      # symmetric
    assert sum(1 for a, b in keys if a == b) == 500                  # diagonal once
    assert len(keys) == g.nnz                                        # no duplicates
    for u in range(0, 500, 37):                                      # ascending per row
        c = g.col_idx[g.row_ptr[u]:g.row_ptr[u + 1]]
        assert np.all(np.diff(c) > 0)


# ---------------------------------------------------------------- G6, Â
def test_dinv_bit_recipe():
    g = oracle.graph_build([0, 0, 0], [1, 2, 3], 5)
    for u in range(5):
        assert g.dinv[u] == np.float32(1.0 / math.sqrt(float(g.deg[u])))


def test_closed_form_edgeless():
    g = oracle.graph_build([], [], 6)
    assert np.array_equal(oracle.a_hat_dense_from_csr(g), np.eye(6))


@pytest.mark.parametrize("n", [2, 5, 9])
def test_closed_form_complete_graph(n):
    iu, ju = np.triu_indices(n, 1)
    g = oracle.graph_build(iu, ju, n)
    assert np.allclose(oracle.a_hat_dense_from_csr(g), np.full((n, n), 1.0 / n), rtol=0, atol=1e-15)


def test_closed_form_regular_cycle():
    n = 11
    src = np.arange(n)
    dst = (src + 1) % n
    g = oracle.graph_build(src, dst, n)
    A = np.zeros((n, n))
    A[src, dst] = A[dst, src] = 1
    assert np.allclose(oracle.a_hat_dense_from_csr(g), (A + np.eye(n)) / 3.0, atol=1e-15)


@pytest.mark.parametrize("leaves", [1, 4, 17])
def test_closed_form_star(leaves):
    n = leaves + 1
    g = oracle.graph_build(np.zeros(leaves, int), np.arange(1, n), n)
    M = oracle.a_hat_dense_from_csr(g)
    assert math.isclose(M[0, 0], 1.0 / (leaves + 1), rel_tol=1e-15)
    assert math.isclose(M[0, 1], 1.0 / math.sqrt(2 * (leaves + 1)), rel_tol=1e-15)
    assert math.isclose(M[1, 1], 0.5, rel_tol=1e-15)
    if leaves > 1:
        assert M[1, 2] == 0.0


def test_row_normalisation_invariants():
    w = make_small(300, 2400, 4, 3, seed=11, alpha=2.1)
    g = oracle.graph_build(w["src"], w["dst"], 300)
    M = oracle.a_hat_dense_from_csr(g)
    sd = np.sqrt(g.deg.astype(np.float64))
    assert np.max(np.abs(M - M.T)) <= 1e-15                                  # Â = Âᵀ
    assert np.max(np.abs(M @ sd - sd)) <= 1e-12                             # Â·√d̃ = √d̃
    P = np.diag(1.0 / g.deg) @ (np.diag(sd) @ M @ np.diag(sd))              # D̃^{-1} Ã
    assert np.max(np.abs(P.sum(axis=1) - 1.0)) <= 1e-14
    ev = np.linalg.eigvalsh(M)
    assert ev.max() <= 1.0 + 1e-12 and ev.min() > -1.0


# ---------------------------------------------------------------- aggregation
@pytest.mark.parametrize("seed,n,m,f", [(0, 40, 100, 3), (1, 300, 3000, 17), (2, 1500, 9000, 33)])
def test_aggregate_vs_dense_definition(seed, n, m, f):
    w = make_small(n, m, f, 3, seed=seed)
    g = oracle.graph_build(w["src"], w["dst"], n)
    X = w["X"].astype(np.float64)
    ref = _dense_a_hat(w["src"], w["dst"], n) @ X
    assert np.max(np.abs(oracle.aggregate(g, X) - ref)) <= 1e-13 * max(1.0, np.abs(ref).max())
    rows = [0, n // 2, n - 1]
    assert np.allclose(oracle.aggregate_rows(g, X, rows), ref[rows], rtol=0, atol=1e-13)


def test_aggregate_identity_and_sqrt_degree():
    g = oracle.graph_build([], [], 7)
    X = np.random.default_rng(0).standard_normal((7, 5))
    assert np.array_equal(oracle.aggregate(g, X), X)
    w = make_small(200, 1000, 2, 2, seed=3)
    g = oracle.graph_build(w["src"], w["dst"], 200)
    sd = np.sqrt(g.deg.astype(np.float64))[:, None] * np.ones((1, 3))
    assert np.allclose(oracle.aggregate(g, sd), sd, rtol=1e-13, atol=0)


def test_aggregate_row_parallel_is_the_same_sum(monkeypatch):
    """The oracle's row-chunked threaded product (c.1: parallel over output rows only) is
    bit-identical to scipy's single-threaded CSR product and matches the one-row-at-a-time
    definition on sampled rows (incl. the largest row)."""
    monkeypatch.setenv("ORACLE_THREADS", "5")
    n = 40_000
    w = make_small(n, 400_000, 9, 4, seed=11)
    g = oracle.graph_build(w["src"], w["dst"], n)
    X = w["X"].astype(np.float64)
    got = oracle.aggregate(g, X)
    import scipy.sparse as sp
    A = sp.csr_matrix((oracle.a_hat_values(g), g.col_idx.astype(np.int64), g.row_ptr), shape=(n, n))
    assert np.array_equal(got, np.asarray(A @ X))
    rows = [0, 1, n // 3, n - 1, int(np.argmax(np.diff(g.row_ptr)))]
    assert np.allclose(got[rows], oracle.aggregate_rows(g, X, rows), rtol=0, atol=1e-13)
    for scheme in ("sum", "mean"):
        for tr in (False, True):
            y = oracle.aggregate_scheme(g, X, scheme, transpose=tr)
            monkeypatch.setenv("ORACLE_THREADS", "1")
            assert np.array_equal(y, oracle.aggregate_scheme(g, X, scheme, transpose=tr))
            monkeypatch.setenv("ORACLE_THREADS", "5")


# ---------------------------------------------------------------- switch S1-S3
def _golden():
    with open(os.path.join(GOLDEN, "paper_constants.json")) as f:
        return json.load(f)


def test_switch_paper_nell_value():
    gd = _golden()
    s_paper = gd["nell_sparsity"]["value"]
    tau_bp = gd["tau"]["tau_bp"]
    n, f = 1000, 1000                       # a NELL-density matrix (0.79 % nonzero)
    X = np.zeros((n, f), np.float32)
    k = int(round((1.0 - s_paper) * n * f))
    X.flat[np.random.default_rng(0).choice(n * f, k, replace=False)] = 1.0
    a = oracle.analyze_features(X, tau_bp)
    assert math.isclose(a.sparsity, s_paper, abs_tol=1e-6)
    assert a.mode == 1 and a.is_binary


def test_switch_boundaries():
    X = np.zeros((10, 10), np.float32)
    X.flat[:20] = 2.5                       # s = 0.80 exactly -> Sparse (inclusive)
    assert oracle.analyze_features(X, 8000).mode == 1
    X.flat[20] = 1.0                        # s = 0.79 -> Dense
    assert oracle.analyze_features(X, 8000).mode == 0
    assert oracle.analyze_features(np.ones((3, 4), np.float32), 8000).mode == 0   # s = 0
    X = np.zeros((4, 4), np.float32)
    X[0, 0] = -0.0                          # -0.0 is zero (Q12)
    assert oracle.analyze_features(X, 8000).nnz == 0
    with pytest.raises(oracle.OracleError):
        oracle.analyze_features(np.zeros((0, 4), np.float32))


def test_switch_monotone_in_sparsity():
    rng = np.random.default_rng(1)
    X = rng.standard_normal((50, 40)).astype(np.float32)
    order = rng.permutation(X.size)
    modes = []
    for k in range(0, X.size + 1, 50):
        Y = X.copy()
        Y.flat[order[:k]] = 0.0
        modes.append(oracle.analyze_features(Y, 8000).mode)
    assert modes == sorted(modes)


def test_csr_csc_round_trip():
    rng = np.random.default_rng(2)
    X = (rng.random((37, 23)) < 0.1).astype(np.float32) * rng.integers(1, 9, (37, 23)).astype(np.float32)
    a = oracle.analyze_features(X, 8000)
    assert a.mode == 1 and not a.is_binary
    ptr, idx, val = a.csr
    D = np.zeros_like(X)
    for i in range(37):
        D[i, idx[ptr[i]:ptr[i + 1]]] = val[ptr[i]:ptr[i + 1]]
    assert np.array_equal(D, X)
    cptr, ridx, cval = a.csc
    E = np.zeros_like(X)
    for k in range(23):
        seg = ridx[cptr[k]:cptr[k + 1]]
        assert np.all(np.diff(seg) > 0)
        E[seg, k] = cval[cptr[k]:cptr[k + 1]]
    assert np.array_equal(E, X)
