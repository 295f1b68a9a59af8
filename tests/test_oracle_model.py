"""Pins for the oracle's model arithmetic: Xavier/splitmix64, Philox dropout,
forward, softmax-CE, backward, Adam and the epoch loop.

Independent references: published known-answer vectors (tests/golden),
closed forms, FP64 central finite differences, and torch.float64 autograd +
torch.optim.Adam on a dense Â built from its definition (an implementation
that shares nothing with oracle/).
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
from synth.generate import make_small, make_sbm_toy

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- Xavier (Q16)
def test_splitmix64_known_answer():
    kat = _load("splitmix64_kat.json")
    out = oracle.splitmix64_stream(kat["seed"], len(kat["outputs_hex"]))
    assert [format(int(x), "016x") for x in out] == kat["outputs_hex"]


def test_xavier_bound_determinism_variance():
    dims = (300, 200, 7)
    W1, b1 = oracle.xavier_init(dims, 42)
    W2, _ = oracle.xavier_init(dims, 42)
    W3, _ = oracle.xavier_init(dims, 43)
    for w, (fi, fo) in zip(W1, [(300, 200), (200, 7)]):
        a = math.sqrt(6.0 / (fi + fo))
        assert w.shape == (fi, fo) and w.dtype == np.float32
        assert np.all(np.abs(w) <= np.float32(a))
    assert all(np.array_equal(a, b) for a, b in zip(W1, W2))
    assert not np.array_equal(W1[0], W3[0])
    var = float(W1[0].astype(np.float64).var())
    assert abs(var - 2.0 / 500) < 0.03 * 2.0 / 500
    assert all(np.all(b == 0) for b in b1)


# ---------------------------------------------------------------- Philox (Q10)
def test_philox_known_answers():
    kat = _load("philox_kat.json")
    for v in kat["vectors"]:
        ctr = np.array([[int(x, 16) for x in v["ctr"]]], dtype=np.uint64)
        key = np.array([[int(x, 16) for x in v["key"]]], dtype=np.uint64)
        out = oracle.philox4x32_10(ctr, key)[0]
        assert [format(int(x), "08x") for x in out] == v["out"]


def test_dropout_keep_rate():
    keep = oracle.dropout_keep(400, 64, 0.3, 12345, 1, 1)
    assert abs(keep.mean() - 0.7) < 0.01
    assert oracle.dropout_keep(10, 8, 0.0, 1, 1, 1).all()
    k2 = oracle.dropout_keep(400, 64, 0.3, 12345, 1, 2)
    assert not np.array_equal(keep, k2)                                     # epoch in counter


# ---------------------------------------------------------------- loss (L1-L3)
def test_loss_uniform_logits_is_log_c():
    for c in (2, 7, 41):
        loss, dZ = oracle.softmax_ce(np.full((5, c), 3.25), np.arange(5) % c)
        assert math.isclose(loss, math.log(c), rel_tol=1e-14)
        assert np.allclose(dZ.sum(axis=1), 0.0, atol=1e-16)


def test_loss_margin_and_logistic():
    Z = np.array([[100.0, 0.0, 0.0]])
    loss, _ = oracle.softmax_ce(Z, [0])
    assert loss < 1e-40
    z = np.array([[0.3, -1.2], [2.0, 0.5]])
    y = np.array([1, 0])
    loss, _ = oracle.softmax_ce(z, y)
    margins = np.array([z[0, 1] - z[0, 0], z[1, 0] - z[1, 1]])
    assert math.isclose(loss, float(np.mean(np.log1p(np.exp(-margins)))), rel_tol=1e-14)


def test_loss_vs_torch_cross_entropy_with_mask():
    rng = np.random.default_rng(0)
    Z = rng.standard_normal((30, 5)) * 4
    y = rng.integers(0, 5, 30)
    mask = rng.random(30) < 0.6
    loss, dZ = oracle.softmax_ce(Z, y, mask)
    tz = torch.tensor(Z, dtype=torch.float64, requires_grad=True)
    ref = torch.nn.functional.cross_entropy(tz[torch.tensor(mask)], torch.tensor(y[mask]))
    ref.backward()
    assert math.isclose(loss, ref.item(), rel_tol=1e-13)
    assert np.allclose(dZ, tz.grad.numpy(), atol=1e-15)


# ---------------------------------------------------------------- forward / backward
def _small_problem(n=16, m=40, dims=(5, 6, 4, 3), seed=0):
    w = make_small(n, m, dims[0], dims[-1], seed=seed)
    g = oracle.graph_build(w["src"], w["dst"], n)
    rng = np.random.default_rng(seed)
    Ws = [rng.standard_normal((dims[i], dims[i + 1])) * 0.7 for i in range(len(dims) - 1)]
    bs = [rng.standard_normal(dims[i + 1]) * 0.1 for i in range(len(dims) - 1)]
    return w, g, Ws, bs


def _loss_of(g, X, y, Ws, bs):
    Z, _ = oracle.forward(g, X, Ws, bs)
    return oracle.softmax_ce(Z, y)[0]


@pytest.mark.parametrize("dims", [(5, 6, 3), (5, 6, 4, 3)])
def test_backward_central_finite_differences(dims):
    w, g, Ws, bs = _small_problem(dims=dims)
    X, y = w["X"].astype(np.float64), w["y"]
    Z, cache = oracle.forward(g, X, Ws, bs)
    _, dZ = oracle.softmax_ce(Z, y)
    dWs, dbs = oracle.backward(g, cache, Ws, dZ)
    h = 1e-6
    pre = [z.copy() for z in cache["Z"][:-1]]
    worst = 0.0
    checked = 0
    for li in range(len(Ws)):
        for arr, grad in ((Ws[li], dWs[li]), (bs[li], dbs[li])):
            for idx in np.ndindex(arr.shape):
                old = arr[idx]
                arr[idx] = old + h
                zp, cp = oracle.forward(g, X, Ws, bs)
                arr[idx] = old - h
                zm, cm = oracle.forward(g, X, Ws, bs)
                arr[idx] = old
                flips = any(np.any(np.sign(a) != np.sign(b)) for a, b in zip(cp["Z"][:-1], pre)) or \
                    any(np.any(np.sign(a) != np.sign(b)) for a, b in zip(cm["Z"][:-1], pre))
                if flips:
                    continue
                fd = (oracle.softmax_ce(zp, y)[0] - oracle.softmax_ce(zm, y)[0]) / (2 * h)
                # FD truncation O(h^2) + rounding ~1e-16/h: relative 1e-6 plus 1e-9 absolute
                err = abs(fd - grad[idx]) / (1e-6 * abs(grad[idx]) + 1e-9)
                worst = max(worst, err)
                checked += 1
    assert checked > 50
    assert worst < 1.0


def _torch_reference(src, dst, n, X, y, Ws, bs, mask=None):
    """Whole forward/backward with torch.float64 autograd on a dense Â from its definition."""
    A = torch.zeros((n, n), dtype=torch.float64)
    for a, b in zip(src.tolist(), dst.tolist()):
        if a != b:
            A[a, b] = 1.0
            A[b, a] = 1.0
    At = A + torch.eye(n, dtype=torch.float64)
    dm = At.sum(1).rsqrt()
    Ah = dm[:, None] * At * dm[None, :]
    tW = [torch.tensor(w, dtype=torch.float64, requires_grad=True) for w in Ws]
    tb = [torch.tensor(b, dtype=torch.float64, requires_grad=True) for b in bs]
    H = torch.tensor(X, dtype=torch.float64)
    for i in range(len(Ws)):
        Z = Ah @ (H @ tW[i]) + tb[i]
        H = torch.relu(Z) if i + 1 < len(Ws) else Z
    yt = torch.tensor(y, dtype=torch.int64)
    if mask is not None:
        mt = torch.tensor(mask)
        loss = torch.nn.functional.cross_entropy(H[mt], yt[mt])
    else:
        loss = torch.nn.functional.cross_entropy(H, yt)
    loss.backward()
    return loss.item(), [w.grad.numpy() for w in tW], [b.grad.numpy() for b in tb], H.detach().numpy()


@pytest.mark.parametrize("seed", [0, 1])
def test_forward_backward_vs_torch_autograd(seed):
    n = 150
    w = make_small(n, 900, 12, 4, seed=seed)
    g = oracle.graph_build(w["src"], w["dst"], n)
    Ws, bs = oracle.xavier_init((12, 16, 8, 4), seed)
    bs = [b + 0.05 for b in bs]
    mask = np.random.default_rng(seed).random(n) < 0.5
    X = w["X"].astype(np.float64)
    Z, cache = oracle.forward(g, X, Ws, bs)
    loss, dZ = oracle.softmax_ce(Z, w["y"], mask)
    dWs, dbs = oracle.backward(g, cache, Ws, dZ)
    rl, rW, rb, rZ = _torch_reference(w["src"], w["dst"], n, X, w["y"], Ws, bs, mask)
    assert np.allclose(Z, rZ, rtol=1e-12, atol=1e-13)
    assert math.isclose(loss, rl, rel_tol=1e-12)
    for a, b in zip(dWs + dbs, rW + rb):
        assert np.allclose(a, b, rtol=1e-10, atol=1e-14)


# ---------------------------------------------------------------- Adam (A1)
def test_adam_first_step_and_zero_grad():
    p = [np.array([1.0, -2.0, 0.5, 3.0])]
    g = [np.array([0.3, -4.0, 0.0, 1e-3])]
    m = [np.zeros(4)]
    v = [np.zeros(4)]
    oracle.adam_step(p, g, m, v, 1, lr=0.01)
    expect = np.array([1.0, -2.0, 0.5, 3.0]) - 0.01 * g[0] / (np.abs(g[0]) + 1e-8)
    assert np.allclose(p[0], expect, rtol=0, atol=1e-15)
    assert p[0][2] == 0.5                                                   # zero grad: no move


def test_adam_constant_gradient_step_tends_to_lr():
    p = [np.zeros(3)]
    m, v = [np.zeros(3)], [np.zeros(3)]
    prev = p[0].copy()
    for t in range(1, 200):
        oracle.adam_step(p, [np.array([0.5, -2.0, 7.0])], m, v, t)
        step = np.abs(p[0] - prev)
        prev = p[0].copy()
    assert np.allclose(step, 0.01, rtol=1e-6)


def test_adam_vs_torch_optim():
    rng = np.random.default_rng(3)
    p0 = rng.standard_normal(20)
    grads = [rng.standard_normal(20) for _ in range(10)]
    p = [p0.copy()]
    m, v = [np.zeros(20)], [np.zeros(20)]
    tp = torch.tensor(p0.copy(), dtype=torch.float64, requires_grad=True)
    opt = torch.optim.Adam([tp], lr=0.01, betas=(0.9, 0.999), eps=1e-8)
    for t, gr in enumerate(grads, 1):
        oracle.adam_step(p, [gr], m, v, t)
        tp.grad = torch.tensor(gr, dtype=torch.float64)
        opt.step()
    assert np.allclose(p[0], tp.detach().numpy(), rtol=0, atol=1e-14)


# ---------------------------------------------------------------- epoch loop
def test_train_matches_torch_for_three_epochs():
    n = 80
    w = make_small(n, 400, 6, 3, seed=7)
    g = oracle.graph_build(w["src"], w["dst"], n)
    dims = (6, 10, 3)
    losses, _ = oracle.train(g, w["X"], w["y"], dims, epochs=3, seed=42)
    Ws, bs = oracle.xavier_init(dims, 42)
    # torch reference of the same loop
    A = torch.zeros((n, n), dtype=torch.float64)
    A[torch.tensor(w["src"], dtype=torch.long), torch.tensor(w["dst"], dtype=torch.long)] = 1.0
    A = ((A + A.T) > 0).double()
    At = A + torch.eye(n, dtype=torch.float64)
    dm = At.sum(1).rsqrt()
    Ah = dm[:, None] * At * dm[None, :]
    tW = [torch.tensor(x, dtype=torch.float64, requires_grad=True) for x in Ws]
    tb = [torch.tensor(x, dtype=torch.float64, requires_grad=True) for x in bs]
    opt = torch.optim.Adam(tW + tb, lr=0.01, betas=(0.9, 0.999), eps=1e-8)
    X = torch.tensor(w["X"], dtype=torch.float64)
    y = torch.tensor(w["y"], dtype=torch.long)
    ref = []
    for _ in range(3):
        opt.zero_grad()
        H = torch.relu(Ah @ (X @ tW[0]) + tb[0])
        Z = Ah @ (H @ tW[1]) + tb[1]
        loss = torch.nn.functional.cross_entropy(Z, y)
        loss.backward()
        ref.append(loss.item())
        opt.step()
    assert np.allclose(losses, ref, rtol=1e-12)


def test_monotone_loss_on_separable_toy():
    w = make_sbm_toy(60, 0.3, 0.02, seed=0)
    g = oracle.graph_build(w["src"], w["dst"], 60)
    losses, params = oracle.train(g, w["X"], w["y"], (2, 16, 2), epochs=200, seed=42)
    assert all(b < a for a, b in zip(losses[:50], losses[1:51]))           # strictly decreasing
    Z, _ = oracle.forward(g, w["X"], params[:2], params[2:])
    assert np.mean(Z.argmax(1) == w["y"]) == 1.0
    losses500, _ = oracle.train(g, w["X"], w["y"], (2, 16, 2), epochs=500, seed=42)
    assert np.all(np.isfinite(losses500))


def test_dropout_forward_backward_fd():
    """With dropout on, the masked network is still differentiable: FD-check a few entries."""
    w, g, Ws, bs = _small_problem(dims=(5, 8, 3), seed=2)
    X, y = w["X"].astype(np.float64), w["y"]
    Z, cache = oracle.forward(g, X, Ws, bs, dropout_p=0.25, seed=99, epoch=3)
    _, dZ = oracle.softmax_ce(Z, y)
    dWs, _ = oracle.backward(g, cache, Ws, dZ)
    h = 1e-6
    for idx in [(0, 0), (2, 3), (4, 7)]:
        old = Ws[0][idx]
        Ws[0][idx] = old + h
        lp = oracle.softmax_ce(oracle.forward(g, X, Ws, bs, 0.25, 99, 3)[0], y)[0]
        Ws[0][idx] = old - h
        lm = oracle.softmax_ce(oracle.forward(g, X, Ws, bs, 0.25, 99, 3)[0], y)[0]
        Ws[0][idx] = old
        fd = (lp - lm) / (2 * h)
        assert abs(fd - dWs[0][idx]) <= 1e-6 * max(1e-3, abs(fd))
