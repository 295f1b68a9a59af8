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


# ---------------------------------------------------------------- TF32 operand rounding (R2)
def test_tf32_rna_known_values():
    """cvt.rna.tf32.f32: 10 explicit mantissa bits, nearest, ties away from zero."""
    u = 2.0 ** -10                                        # TF32 ulp at 1.0
    cases = {1.0: 1.0, 1.0 + u / 2: 1.0 + u, -(1.0 + u / 2): -(1.0 + u), 1.0 + u / 4: 1.0,
             1.0 + 3 * u / 4: 1.0 + u, 1.0 + u + u / 2: 1.0 + 2 * u, 3.0 * 2.0 ** 100: 3.0 * 2.0 ** 100,
             0.0: 0.0, 2.0 - u / 2: 2.0, 1.0 + 2.0 ** -23: 1.0}
    for x, want in cases.items():
        assert oracle.tf32_rna(np.float32(x)) == want, x
    # subnormal fp32 input: same rule on the raw mantissa
    sub = np.array([0x00001000], np.uint32).view(np.float32)
    assert oracle.tf32_rna(sub).item() == np.array([0x00002000], np.uint32).view(np.float32).item()


def test_tf32_rna_properties():
    rng = np.random.default_rng(0)
    x = (rng.standard_normal(100000) * np.exp(rng.uniform(-20, 20, 100000))).astype(np.float32)
    r = oracle.tf32_rna(x)
    assert np.all(np.abs(r - x) <= 2.0 ** -11 * np.abs(x.astype(np.float64)))
    assert np.all(r.astype(np.float32).view(np.uint32) & 0x1FFF == 0)
    assert np.array_equal(oracle.tf32_rna(r), r)                  # idempotent
    assert np.array_equal(oracle.tf32_rna(-x), -r)                # symmetric (ties away from zero)


def test_tf32_forward_within_operand_bound():
    """operand_rounding="tf32" changes each dense product H·W by at most (2^-11 + 2^-11 + 2^-22)|H||W|
    per element before aggregation; Â is nonnegative, so Z moves by at most Â(that bound)."""
    w = make_small(300, 2400, 24, 5, seed=5)
    g = oracle.graph_build(w["src"], w["dst"], 300)
    dims = (24, 16, 5)
    Ws, bs = oracle.xavier_init(dims, 42)
    Z0, c0 = oracle.forward(g, w["X"], Ws, bs)
    Z1, c1 = oracle.forward(g, w["X"], Ws, bs, operand_rounding="tf32")
    e = 2.0 ** -11 * 2 + 2.0 ** -22
    b1 = oracle.aggregate(g, e * np.abs(w["X"].astype(np.float64)) @ np.abs(Ws[0].astype(np.float64)))
    z1_exact = c0["Z"][0]
    assert np.all(np.abs(c1["Z"][0] - z1_exact) <= b1 + 1e-15)
    assert not np.array_equal(c1["Z"][0], z1_exact)               # the option does something
    # sparse X: the layer-1 product stays exact
    _, cs = oracle.forward(g, sp.csr_matrix(w["X"]), Ws, bs, operand_rounding="tf32")
    assert np.allclose(cs["Z"][0], z1_exact, rtol=1e-13, atol=1e-15)


# ---------------------------------------------------------------- BF16 operand rounding (north star option)
def test_bf16_rne_known_values():
    """cvt.rn.bf16.f32: 7 explicit mantissa bits, nearest, ties to even."""
    u = 2.0 ** -7                                         # BF16 ulp at 1.0
    cases = {1.0: 1.0, 1.0 + u / 2: 1.0, 1.0 + u + u / 2: 1.0 + 2 * u, -(1.0 + u + u / 2): -(1.0 + 2 * u),
             1.0 + u / 4: 1.0, 1.0 + 3 * u / 4: 1.0 + u, 2.0 - u / 4: 2.0, 0.0: 0.0,
             3.0 * 2.0 ** 100: 3.0 * 2.0 ** 100, 1.0 + 2.0 ** -23: 1.0}
    for x, want in cases.items():
        assert oracle.bf16_rne(np.float32(x)) == want, x


def test_bf16_rne_properties_and_torch():
    import torch
    rng = np.random.default_rng(1)
    x = (rng.standard_normal(100000) * np.exp(rng.uniform(-20, 20, 100000))).astype(np.float32)
    r = oracle.bf16_rne(x)
    assert np.all(np.abs(r - x) <= 2.0 ** -8 * np.abs(x.astype(np.float64)))
    assert np.all(r.astype(np.float32).view(np.uint32) & 0xFFFF == 0)
    assert np.array_equal(oracle.bf16_rne(r), r)                   # idempotent
    assert np.array_equal(oracle.bf16_rne(-x), -r)                 # symmetric
    # an independent implementation of the same rounding: torch's float32 -> bfloat16 cast
    t = torch.from_numpy(x).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(r, t)


def test_bf16_trajectory_within_north_star():
    """BF16 GEMM operands (each dense product's operands rounded by bf16_rne, FP32-exact
    accumulation in the oracle) keep loss_1..loss_10 within the north star's 1e-3 of the exact
    trajectory on a Pubmed-shaped graph forced dense — the accuracy case for a BF16 path."""
    w = make_small(2000, 16000, 60, 3, kind="dense", seed=11, alpha=2.4, mu=0.2)
    g = oracle.graph_build(w["src"], w["dst"], 2000)
    dims = (60, 32, 3)
    ex, _ = oracle.train(g, w["X"], w["y"], dims, epochs=10, seed=42)
    bf, _ = oracle.train(g, w["X"], w["y"], dims, epochs=10, seed=42, operand_rounding="bf16")
    ex, bf = np.array(ex), np.array(bf)
    assert np.all(np.abs(bf - ex) <= 1e-3 * np.maximum(1.0, np.abs(ex))), np.abs(bf - ex).max()
    assert not np.array_equal(bf, ex)


# ---------------------------------------------------------------- layer order (reading Q7)
def test_aggregate_first_equals_transform_first_exact():
    """orders=("AF", ...) computes Z = (Â·H)·W + b instead of Â·(H·W) + b: the same numbers in
    exact arithmetic (associativity of the linear maps), so without operand rounding the
    loss and every gradient agree to FP64 rounding, for the GCN and the linear schemes (mean is
    not symmetric, so its AF backward needs the adjoint D̃⁻¹-on-the-right path to be right)."""
    w = make_small(400, 3200, 12, 4, seed=8)
    g = oracle.graph_build(w["src"], w["dst"], 400)
    dims = (12, 20, 16, 4)
    Ws, bs = oracle.xavier_init(dims, 42)
    for agg in ("gcn", "sum", "mean"):
        Zt, ct = oracle.forward(g, w["X"], Ws, bs, aggregator=agg)
        Za, ca = oracle.forward(g, w["X"], Ws, bs, aggregator=agg, orders=("AF", "AF", "TF"))
        assert np.allclose(Za, Zt, rtol=1e-12, atol=1e-12)
        lt, dZt = oracle.softmax_ce(Zt, w["y"])
        la, dZa = oracle.softmax_ce(Za, w["y"])
        assert abs(lt - la) <= 1e-12 * abs(lt)
        gt = oracle.backward(g, ct, Ws, dZt)
        ga = oracle.backward(g, ca, Ws, dZa)
        for a, b in zip(gt[0] + gt[1], ga[0] + ga[1]):
            assert np.allclose(a, b, rtol=1e-10, atol=1e-14), agg


def test_aggregate_first_gradient_by_finite_differences():
    """An independent pin of the AF backward (not a re-derivation of it): central differences of
    the loss in three entries of W_1 and b_1 of an aggregate-first layer 1."""
    w = make_small(120, 700, 6, 3, seed=9)
    g = oracle.graph_build(w["src"], w["dst"], 120)
    dims = (6, 9, 3)
    Ws, bs = [np.asarray(a, np.float64) for a in oracle.xavier_init(dims, 3)[0]], \
        [np.asarray(b, np.float64) + 0.01 for b in oracle.xavier_init(dims, 3)[1]]
    orders = ("AF", "TF")
    Z, c = oracle.forward(g, w["X"], Ws, bs, orders=orders)
    _, dZ = oracle.softmax_ce(Z, w["y"])
    dW, db = oracle.backward(g, c, Ws, dZ)

    def loss_at(Wm, bm):
        return oracle.softmax_ce(oracle.forward(g, w["X"], Wm, bm, orders=orders)[0], w["y"])[0]
    h = 1e-6
    for (i, j) in ((0, 0), (3, 5), (5, 8)):
        Wp = [a.copy() for a in Ws]
        Wm = [a.copy() for a in Ws]
        Wp[0][i, j] += h
        Wm[0][i, j] -= h
        fd = (loss_at(Wp, bs) - loss_at(Wm, bs)) / (2 * h)
        assert abs(fd - dW[0][i, j]) <= 1e-6 * max(1.0, abs(fd)), (i, j, fd, dW[0][i, j])
    bp = [b.copy() for b in bs]
    bm = [b.copy() for b in bs]
    bp[0][2] += h
    bm[0][2] -= h
    fd = (loss_at(Ws, bp) - loss_at(Ws, bm)) / (2 * h)
    assert abs(fd - db[0][2]) <= 1e-6 * max(1.0, abs(fd))


def test_tf32_aggregate_first_rounds_the_aggregate():
    """With operand_rounding="tf32", an AF layer 1 rounds Y = Â·X (the kernel's stored operand)
    and not X: Z_1 moves from the exact value by at most (2^-11 + 2^-11 + 2^-22)|Y||W| (the GEMM
    bound of one rounded product), and differs from the TF-rounded Z_1."""
    w = make_small(300, 2400, 24, 5, seed=5)
    g = oracle.graph_build(w["src"], w["dst"], 300)
    dims = (24, 40, 5)
    Ws, bs = oracle.xavier_init(dims, 42)
    _, c0 = oracle.forward(g, w["X"], Ws, bs)
    _, ca = oracle.forward(g, w["X"], Ws, bs, operand_rounding="tf32", orders=("AF", "TF"))
    _, ct = oracle.forward(g, w["X"], Ws, bs, operand_rounding="tf32")
    Y = oracle.aggregate(g, w["X"].astype(np.float64))
    e = 2.0 ** -11 * 2 + 2.0 ** -22
    assert np.all(np.abs(ca["Z"][0] - c0["Z"][0]) <= e * np.abs(Y) @ np.abs(Ws[0].astype(np.float64)) + 1e-15)
    assert not np.array_equal(ca["Z"][0], ct["Z"][0])
    assert np.array_equal(ca["Y"][0], Y)
