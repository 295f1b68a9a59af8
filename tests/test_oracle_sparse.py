"""Pins for the oracle's CSR-feature path (NELL-scale inputs): the sparse
branch of analyze_features and of forward/backward must equal the dense branch (which is itself
pinned in test_oracle_graph / test_oracle_model) on the same matrix, and the synthetic NELL
features must carry the paper's sparsity."""
import json
import os

import numpy as np
import scipy.sparse as sp

import oracle
from synth.generate import make_features_csr, make_labels, make_small

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_sparse_and_dense_feature_analysis_agree():
    rng = np.random.default_rng(0)
    X = (rng.random((300, 97)) < 0.08).astype(np.float32) * rng.integers(1, 5, (300, 97)).astype(np.float32)
    Xs = sp.csr_matrix(X)
    for tau in (8000, 9500):
        a, b = oracle.analyze_features(X, tau), oracle.analyze_features(Xs, tau)
        assert (a.nnz, a.mode, a.is_binary) == (b.nnz, b.mode, b.is_binary)
        if a.mode == 1:
            for u, v in zip(a.csr + a.csc, b.csr + b.csc):
                assert np.array_equal(u, v)


def test_sparse_and_dense_training_agree():
    w = make_small(200, 1400, 64, 4, kind="binary", density=0.05, seed=3)
    g = oracle.graph_build(w["src"], w["dst"], 200)
    la, pa = oracle.train(g, w["X"], w["y"], (64, 16, 4), epochs=3, seed=42)
    lb, pb = oracle.train(g, sp.csr_matrix(w["X"]), w["y"], (64, 16, 4), epochs=3, seed=42)
    assert np.allclose(la, lb, rtol=1e-13)
    assert all(np.allclose(x, y, rtol=1e-12, atol=1e-15) for x, y in zip(pa, pb))


def test_nell_features_have_the_papers_sparsity():
    with open(os.path.join(GOLDEN, "paper_constants.json")) as f:
        gd = json.load(f)
    n, fdim = gd["nell_shape"]["num_nodes"], gd["nell_shape"]["num_features"]
    c = 186
    y = make_labels(n, c)
    ptr, idx, val = make_features_csr(n, fdim, y, c, 1.0 - gd["nell_sparsity"]["value"], seed=6)
    s = 1.0 - val.size / (n * fdim)
    assert abs(s - gd["nell_sparsity"]["value"]) < 2e-4
    assert np.all(np.diff(ptr) >= 0) and ptr[-1] == val.size
    Xs = sp.csr_matrix((val, idx, ptr), shape=(n, fdim))
    a = oracle.analyze_features(Xs, gd["tau"]["tau_bp"])
    assert a.mode == 1 and a.is_binary and a.nnz == val.size
