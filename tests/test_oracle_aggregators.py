"""Pins for the oracle's other aggregation schemes and optimizers (P:99,
P:140; readings R6-R8 in DESIGN.md).  Each scheme is pinned to
something other than itself: a brute-force loop over the neighbour sets built from the raw edge
list, finite differences of the whole training loss, torch.float64 autograd on dense matrices
written from the definition, torch.optim for the optimizers, and tiny hand cases."""
import math

import numpy as np
import pytest
import torch

import oracle
from synth.generate import make_sbm_toy, make_small


def _neighbour_sets(src, dst, n):
    """Ñ(u) = N(u) ∪ {u} from the raw (possibly duplicated / self-looped) edge list (Q2-Q4, R6)."""
    nb = [{u} for u in range(n)]
    for a, b in zip(src.tolist(), dst.tolist()):
        nb[a].add(b)
        nb[b].add(a)
    return [sorted(s) for s in nb]


def _graph(n=30, m=80, seed=0):
    w = make_small(n, m, 4, 3, seed=seed)
    return w, oracle.graph_build(w["src"], w["dst"], n), _neighbour_sets(w["src"], w["dst"], n)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_linear_schemes_brute_force(seed):
    w, g, nb = _graph(seed=seed)
    n = g.num_nodes
    P = np.random.default_rng(seed).standard_normal((n, 5))
    sum_ref = np.array([[sum(P[v, c] for v in nb[u]) for c in range(5)] for u in range(n)])
    mean_ref = np.array([[sum(P[v, c] for v in nb[u]) / len(nb[u]) for c in range(5)] for u in range(n)])
    gcn_ref = np.array([[sum(P[v, c] / math.sqrt(len(nb[u]) * len(nb[v])) for v in nb[u]) for c in range(5)]
                        for u in range(n)])
    assert np.allclose(oracle.aggregate_scheme(g, P, "sum"), sum_ref, rtol=1e-14, atol=1e-14)
    assert np.allclose(oracle.aggregate_scheme(g, P, "mean"), mean_ref, rtol=1e-14, atol=1e-14)
    assert np.allclose(oracle.aggregate_scheme(g, P, "gcn"), gcn_ref, rtol=1e-13, atol=1e-14)
    # adjoints from the dense matrices of the definitions
    M = np.zeros((n, n))
    for u in range(n):
        for v in nb[u]:
            M[u, v] = 1.0 / len(nb[u])
    assert np.allclose(oracle.aggregate_scheme(g, P, "mean", transpose=True), M.T @ P, rtol=1e-13, atol=1e-14)
    S = (M > 0).astype(float)
    assert np.allclose(oracle.aggregate_scheme(g, P, "sum", transpose=True), S.T @ P, rtol=1e-14, atol=1e-14)


def test_linear_scheme_invariants():
    w, g, nb = _graph(60, 200, seed=4)
    n = g.num_nodes
    ones = np.ones((n, 1))
    assert np.array_equal(oracle.aggregate_scheme(g, ones, "sum")[:, 0], g.deg.astype(float))   # Ã·1 = d̃
    c = np.full((n, 3), 2.5)
    assert np.allclose(oracle.aggregate_scheme(g, c, "mean"), c, rtol=1e-15)                 # mean of a constant
    # isolated node (no edges): every scheme returns its own row (self loop only, R6)
    gi = oracle.graph_build(np.array([0], np.int32), np.array([1], np.int32), 3)
    P = np.array([[1.0, -2.0], [3.0, 4.0], [5.0, -6.0]])
    for s in ("sum", "mean", "gcn"):
        assert np.array_equal(oracle.aggregate_scheme(gi, P, s)[2], P[2])
    Y, arg = oracle.aggregate_max(gi, P)
    assert np.array_equal(Y[2], P[2]) and np.all(arg[2] == 2)


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_max_brute_force_with_ties(seed):
    """Integer-valued features make ties common: the smallest neighbour id must win (R7)."""
    w, g, nb = _graph(40, 120, seed=seed)
    n = g.num_nodes
    P = np.random.default_rng(seed).integers(0, 3, (n, 6)).astype(np.float64)
    Y, arg = oracle.aggregate_max(g, P)
    for u in range(n):
        for c in range(6):
            best, bv = None, -np.inf
            for v in nb[u]:                       # ascending ids; strict > keeps the first maximum
                if P[v, c] > bv:
                    best, bv = v, P[v, c]
            assert Y[u, c] == bv and arg[u, c] == best


def test_max_tie_hand_case():
    # star: centre 3 joined to 0, 1, 2, 4; leaves 1 and 4 tie with the centre at 7
    src = np.array([3, 3, 3, 3], np.int32)
    dst = np.array([0, 1, 2, 4], np.int32)
    g = oracle.graph_build(src, dst, 5)
    P = np.array([[1.0], [7.0], [2.0], [7.0], [7.0]])
    Y, arg = oracle.aggregate_max(g, P)
    assert Y[3, 0] == 7.0 and arg[3, 0] == 1     # smallest of {1, 3, 4}
    assert arg[0, 0] == 3 and arg[4, 0] == 3     # leaf 4: {3, 4} tie -> 3
    dH = oracle.aggregate_max_backward(np.ones((5, 1)), arg, 5)
    # arg = [3, 1, 3, 1, 3] (node 1: {1, 3} tie -> 1; node 2: {2, 3} -> 3): node 1 receives from
    # u = 1, 3 and node 3 from u = 0, 2, 4
    assert arg[:, 0].tolist() == [3, 1, 3, 1, 3]
    assert dH[:, 0].tolist() == [0.0, 2.0, 0.0, 3.0, 0.0]


def test_max_backward_is_the_derivative():
    """sum(Y ⊙ R) is piecewise linear in P; away from ties its exact derivative is the
    routing adjoint (checked by central differences) and the routed mass is conserved."""
    w, g, _ = _graph(50, 150, seed=5)
    rng = np.random.default_rng(5)
    P = rng.standard_normal((50, 4))
    R = rng.standard_normal((50, 4))
    Y, arg = oracle.aggregate_max(g, P)
    dP = oracle.aggregate_max_backward(R, arg, 50)
    assert np.allclose(dP.sum(0), R.sum(0), rtol=1e-13)
    h = 1e-7
    for v in range(50):
        for c in range(4):
            Pp, Pm = P.copy(), P.copy()
            Pp[v, c] += h
            Pm[v, c] -= h
            fd = ((oracle.aggregate_max(g, Pp)[0] * R).sum() - (oracle.aggregate_max(g, Pm)[0] * R).sum()) / (2 * h)
            assert abs(fd - dP[v, c]) <= 1e-6 * (1 + abs(dP[v, c]))


@pytest.mark.parametrize("agg", ["sum", "mean", "max"])
@pytest.mark.parametrize("dims", [(5, 6, 3), (5, 6, 4, 3)])
def test_backward_central_finite_differences_all_schemes(agg, dims):
    w = make_small(16, 40, dims[0], dims[-1], seed=1)
    g = oracle.graph_build(w["src"], w["dst"], 16)
    rng = np.random.default_rng(1)
    Ws = [rng.standard_normal((dims[i], dims[i + 1])) * 0.7 for i in range(len(dims) - 1)]
    bs = [rng.standard_normal(dims[i + 1]) * 0.1 for i in range(len(dims) - 1)]
    X, y = w["X"].astype(np.float64) + rng.standard_normal(w["X"].shape) * 0.01, w["y"]   # generic: no max ties
    Z, cache = oracle.forward(g, X, Ws, bs, aggregator=agg)
    _, dZ = oracle.softmax_ce(Z, y)
    dWs, dbs = oracle.backward(g, cache, Ws, dZ)
    h = 1e-6
    worst, checked = 0.0, 0
    for li in range(len(Ws)):
        for arr, grad in ((Ws[li], dWs[li]), (bs[li], dbs[li])):
            for idx in np.ndindex(arr.shape):
                old = arr[idx]
                arr[idx] = old + h
                zp, cp = oracle.forward(g, X, Ws, bs, aggregator=agg)
                arr[idx] = old - h
                zm, cm = oracle.forward(g, X, Ws, bs, aggregator=agg)
                arr[idx] = old
                kink = any(np.any(np.sign(a) != np.sign(b)) for c2 in (cp, cm) for a, b in zip(c2["Z"][:-1], cache["Z"][:-1]))
                if agg == "max":
                    kink = kink or any(np.any(a != b) for c2 in (cp, cm) for a, b in zip(c2["arg"], cache["arg"]))
                if kink:
                    continue
                fd = (oracle.softmax_ce(zp, y)[0] - oracle.softmax_ce(zm, y)[0]) / (2 * h)
                worst = max(worst, abs(fd - grad[idx]) / (1e-6 * abs(grad[idx]) + 1e-9))
                checked += 1
    assert checked > 40
    assert worst < 1.0


@pytest.mark.parametrize("agg", ["sum", "mean"])
def test_linear_schemes_vs_torch_autograd(agg):
    n = 120
    w = make_small(n, 700, 10, 4, seed=9)
    g = oracle.graph_build(w["src"], w["dst"], n)
    nb = _neighbour_sets(w["src"], w["dst"], n)
    M = torch.zeros((n, n), dtype=torch.float64)
    for u in range(n):
        for v in nb[u]:
            M[u, v] = 1.0 / len(nb[u]) if agg == "mean" else 1.0
    Ws, bs = oracle.xavier_init((10, 12, 4), 3)
    bs = [b + 0.05 for b in bs]
    X = w["X"].astype(np.float64)
    Z, cache = oracle.forward(g, X, Ws, bs, aggregator=agg)
    loss, dZ = oracle.softmax_ce(Z, w["y"])
    dWs, dbs = oracle.backward(g, cache, Ws, dZ)
    tW = [torch.tensor(x, dtype=torch.float64, requires_grad=True) for x in Ws]
    tb = [torch.tensor(x, dtype=torch.float64, requires_grad=True) for x in bs]
    H = torch.tensor(X)
    for i in range(2):
        Zt = M @ (H @ tW[i]) + tb[i]
        H = torch.relu(Zt) if i == 0 else Zt
    lt = torch.nn.functional.cross_entropy(H, torch.tensor(w["y"], dtype=torch.long))
    lt.backward()
    assert math.isclose(loss, lt.item(), rel_tol=1e-12)
    for a, b in zip(dWs + dbs, [x.grad.numpy() for x in tW + tb]):
        assert np.allclose(a, b, rtol=1e-10, atol=1e-14)


# ---------------------------------------------------------------- optimizers
def test_sgd_closed_forms():
    p = [np.array([1.0, -2.0])]
    oracle.sgd_step(p, [np.array([0.5, 4.0])], [np.zeros(2)], lr=0.1)
    assert np.allclose(p[0], [0.95, -2.4], rtol=0, atol=1e-15)
    p, vel = [np.array([1.0])], [np.zeros(1)]
    oracle.sgd_step(p, [np.array([2.0])], vel, lr=0.1, momentum=0.9)      # v = 2,   p = 0.8
    oracle.sgd_step(p, [np.array([2.0])], vel, lr=0.1, momentum=0.9)      # v = 3.8, p = 0.42
    assert abs(p[0][0] - 0.42) < 1e-15 and abs(vel[0][0] - 3.8) < 1e-15


@pytest.mark.parametrize("momentum,wd", [(0.0, 0.0), (0.9, 0.0), (0.9, 0.01), (0.0, 0.05)])
def test_sgd_vs_torch_optim(momentum, wd):
    rng = np.random.default_rng(4)
    p0 = rng.standard_normal(30)
    p, vel = [p0.copy()], [np.zeros(30)]
    tp = torch.tensor(p0.copy(), dtype=torch.float64, requires_grad=True)
    opt = torch.optim.SGD([tp], lr=0.05, momentum=momentum, weight_decay=wd)
    for _ in range(8):
        gr = rng.standard_normal(30)
        oracle.sgd_step(p, [gr], vel, lr=0.05, momentum=momentum, weight_decay=wd)
        tp.grad = torch.tensor(gr, dtype=torch.float64)
        opt.step()
    assert np.allclose(p[0], tp.detach().numpy(), rtol=0, atol=1e-14)


def test_adamw_vs_torch_optim_and_decoupling():
    rng = np.random.default_rng(6)
    p0 = rng.standard_normal(25)
    p, m, v = [p0.copy()], [np.zeros(25)], [np.zeros(25)]
    tp = torch.tensor(p0.copy(), dtype=torch.float64, requires_grad=True)
    opt = torch.optim.AdamW([tp], lr=0.01, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.05)
    for t in range(1, 11):
        gr = rng.standard_normal(25)
        oracle.adamw_step(p, [gr], m, v, t, weight_decay=0.05)
        tp.grad = torch.tensor(gr, dtype=torch.float64)
        opt.step()
    assert np.allclose(p[0], tp.detach().numpy(), rtol=0, atol=1e-14)
    # zero gradient: only the decay acts (decoupled: it never enters m or v)
    q, mq, vq = [np.array([2.0, -1.0])], [np.zeros(2)], [np.zeros(2)]
    oracle.adamw_step(q, [np.zeros(2)], mq, vq, 1, lr=0.1, weight_decay=0.5)
    assert np.allclose(q[0], [1.9, -0.95], rtol=0, atol=1e-15) and not mq[0].any() and not vq[0].any()


@pytest.mark.parametrize("agg", ["sum", "mean", "max"])
@pytest.mark.parametrize("opt", ["adam", "sgd", "adamw"])
def test_training_learns_the_separable_toy(agg, opt):
    w = make_sbm_toy(60, 0.3, 0.02, seed=0)
    g = oracle.graph_build(w["src"], w["dst"], 60)
    kw = {"lr": 0.01, "momentum": 0.9} if opt == "sgd" else {"weight_decay": 0.01} if opt == "adamw" else {}
    losses, params = oracle.train(g, w["X"], w["y"], (2, 16, 2), epochs=150, seed=42, aggregator=agg,
                                  optimizer=opt, **kw)
    assert np.all(np.isfinite(losses)) and losses[-1] < 0.5 * losses[0]
    Z, _ = oracle.forward(g, w["X"], params[:2], params[2:], aggregator=agg)
    assert np.mean(Z.argmax(1) == w["y"]) >= 0.95
