"""Parity at BASELINE.json's full sizes (Reddit- and ogbn-products-shaped), in the launch
configuration bench.py times, on sampled outputs the oracle computes one by one, plus
properties that hold at any size (③ of the task).

* a0: nnz exact, sampled CSR rows bit-equal the edge list's neighbourhoods (+ self), dinv
  bit recipe on every row.
* a2/a3: for sampled rows (incl. the two largest hubs), H_1[u] = relu((Â·X·W_1)[u] + b_1)
  within the TF32 GEMM bound composed through the aggregation.
* epoch-1 loss (forward at θ_0) against the full FP64 oracle's (golden, tools/make_goldens.py);
  the 10-epoch trajectories, gradients and BF16 runs are in test_gpu_fullsize_train.py.
* a3 at full hub degree: the 64 largest Reddit hubs within the FP32 aggregation bar.
"""
import ctypes as C
import math

import numpy as np
import pytest
import torch

import oracle
from synth.generate import make_workload

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

SAMPLE_ROWS = 48


@pytest.fixture(scope="module")
def P():
    import paper_2512_01678_b200 as P
    from paper_2512_01678_b200 import _lib as L
    L.mph_device_check(C.byref(C.c_int32()))
    return P


def _neighbourhood(src, dst, u):
    nb = np.concatenate([dst[src == u], src[dst == u], [u]])
    return np.unique(nb)


def _model(P, w):
    cfg = w["cfg"]
    g = P.Graph(w["src"], w["dst"], cfg.num_nodes)
    f = P.Features(torch.from_numpy(w["X"]).cuda())
    m = P.GCN(g, f, cfg.dims)
    m.init_xavier(42)
    m.set_labels(torch.from_numpy(w["y"]).cuda())
    return g, f, m


def _check_graph(g, w, rows):
    """Whole CSR bit-exact against the oracle's own build, plus sampled neighbourhoods."""
    cfg = w["cfg"]
    assert g.nnz == cfg.nnz_a + cfg.num_nodes
    rp, ci, dg, di = g.csr()
    rp = rp.cpu().numpy()
    assert np.all(np.diff(rp) >= 1) and rp[0] == 0 and rp[-1] == g.nnz
    deg = np.diff(rp)
    assert np.array_equal(dg.cpu().numpy(), deg)
    dref = (1.0 / np.sqrt(deg.astype(np.float64))).astype(np.float32)
    assert np.array_equal(di.cpu().numpy().view(np.uint32), dref.view(np.uint32))
    ci = ci.cpu().numpy()
    for u in rows:
        assert np.array_equal(ci[rp[u]:rp[u + 1]], _neighbourhood(w["src"], w["dst"], u)), f"row {u}"
    ref = oracle.graph_build(w["src"], w["dst"], cfg.num_nodes)
    assert np.array_equal(rp, ref.row_ptr) and np.array_equal(ci, ref.col_idx)
    return ref, rp, ci, di.cpu().numpy()


def _check_layer1_tf(m, w, ref_g, rows):
    """Reddit layer 1 (transform-first) on sampled rows.  Expected values come from the oracle
    only (X, Xavier W_1 and the oracle's own CSR); the bound composes the TF32 GEMM tolerance
    through the aggregation, plus half a TF32 ulp for the stored H_1."""
    m.forward(1)
    torch.cuda.synchronize()
    Ws, _ = oracle.xavier_init(w["cfg"].dims, 42)
    W1 = Ws[0].astype(np.float64)
    H1 = m.tensor(1, 1).cpu().numpy()
    X = w["X"]
    d = ref_g.deg.astype(np.float64)
    for u in rows:
        nb = ref_g.col_idx[ref_g.row_ptr[u]:ref_g.row_ptr[u + 1]].astype(np.int64)
        a = 1.0 / np.sqrt(d[u] * d[nb])                       # â_uv (Q1)
        Xn = X[nb].astype(np.float64)
        z = a @ (Xn @ W1)                                      # b_1 = 0 at θ_0
        bound = a @ (np.abs(Xn) @ np.abs(W1))
        lim = 2e-3 * bound + 2.0 ** -11 * np.abs(z) + 1e-30
        assert np.all(np.abs(H1[u] - np.maximum(z, 0)) <= lim), f"H1 row {u}"


def _golden_loss1(name):
    """loss_1 of the FP64 oracle at full size (tests/golden, written by tools/make_goldens.py)."""
    import os
    return float(np.load(os.path.join(os.path.dirname(__file__), "golden", f"fullsize_{name}.npz"))["losses"][0])


@pytest.fixture(scope="module")
def reddit():
    return make_workload("reddit")


def test_reddit_graph_layer1_and_loss(P, reddit):
    w = reddit
    rng = np.random.default_rng(0)
    n = w["cfg"].num_nodes
    g, f, m = _model(P, w)
    rows = list(rng.choice(n, SAMPLE_ROWS - 2, replace=False))
    ref_g, rp, ci, dinv = _check_graph(g, w, rows)
    rows += list(np.argsort(np.diff(rp))[-2:])       # the two largest hubs
    _check_layer1_tf(m, w, ref_g, rows)
    loss = m.loss().item()
    torch.cuda.synchronize()
    ref_loss = _golden_loss1("reddit")
    assert abs(loss - ref_loss) <= 1e-3 * max(1.0, abs(ref_loss)), (loss, ref_loss)


@pytest.fixture(scope="module")
def reddit_graphs(P, reddit):
    w = reddit
    n = w["cfg"].num_nodes
    return P.Graph(w["src"], w["dst"], n), oracle.graph_build(w["src"], w["dst"], n)


@pytest.mark.parametrize("w", [48, 64, 128])
def test_reddit_hub_rows_spmm(P, reddit_graphs, w):
    """The FP32 aggregation bar 1e-5·(|Â|·|T|) on the full Reddit-shaped graph's 64 largest hubs
    (degrees up to ~9.5K, where a single running FP32 sum would exceed the bar: SURVEY c.5's
    accumulation budget, ⌈deg/256⌉ partial sums) plus 64 random rows, in the launch
    configuration the epoch uses for each width (w = 128 runs as two 64-wide column slabs).
    Expected values: the oracle's one-row-at-a-time Â·T on the same FP32 inputs."""
    g, ref = reddit_graphs
    n = ref.num_nodes
    deg = np.diff(ref.row_ptr)
    hubs = np.argsort(deg, kind="stable")[-64:]
    rng = np.random.default_rng(1000 + w)
    rows = np.concatenate([hubs, rng.choice(n, 64, replace=False)])
    print(f"hub degrees {int(deg[hubs].min())}..{int(deg[hubs].max())}")
    assert deg[hubs].max() > 9000
    T = rng.standard_normal((n, w)).astype(np.float32)
    Tp = (ref.dinv[:, None] * T).astype(np.float32)
    out = torch.zeros((n, w), device="cuda")
    g.spmm(torch.from_numpy(Tp).cuda(), out, w=w)
    Z = out.cpu().numpy()[rows]
    Zref = oracle.aggregate_rows(ref, T, rows)
    bound = oracle.aggregate_rows(ref, np.abs(T), rows)
    err = np.abs(Z.astype(np.float64) - Zref)
    ratio = float((err / (1e-5 * bound + 1e-30)).max())
    print(f"w={w}: max |err|/(1e-5·|Â||T|) = {ratio:.3g} (hubs {float((err[:64] / (1e-5 * bound[:64])).max()):.3g})")
    assert ratio <= 1.0


@pytest.fixture(scope="module")
def products_graphs(P):
    w = make_workload("products")
    n = w["cfg"].num_nodes
    return P.Graph(w["src"], w["dst"], n), oracle.graph_build(w["src"], w["dst"], n)


@pytest.mark.parametrize("w", [48, 104, 128, 256])
def test_products_hub_rows_spmm(P, products_graphs, w):
    """The FP32 aggregation bar 1e-5·(|Â|·|T|) on the full products-shaped graph's 64 largest hubs
    (degrees up to ~7.5K) plus 64 random rows, in the launch configuration the epoch uses: w = 104
    and 128 walk the chunked virtual CSR (hub rows cut into chunks of 256 edges whose partial rows
    k_spmm_combine adds in chunk order), w = 256 as two such 128-wide slabs, w = 48
    the hub-first whole-row items.  Expected values: the oracle's one-row-at-a-time Â·T."""
    g, ref = products_graphs
    n = ref.num_nodes
    deg = np.diff(ref.row_ptr)
    hubs = np.argsort(deg, kind="stable")[-64:]
    rng = np.random.default_rng(2000 + w)
    rows = np.concatenate([hubs, rng.choice(n, 64, replace=False)])
    assert deg[hubs].max() > 5000 and deg[hubs].min() > 256   # every hub is cut into chunks
    T = rng.standard_normal((n, w)).astype(np.float32)
    Tp = (ref.dinv[:, None] * T).astype(np.float32)
    out = torch.zeros((n, w), device="cuda")
    tin = torch.from_numpy(Tp).cuda()
    g.spmm(tin, out, w=w)
    out2 = torch.zeros_like(out)
    g.spmm(tin, out2, w=w)
    torch.cuda.synchronize()
    assert torch.equal(out, out2)   # deterministic whatever order the chunks ran in
    Z = out.cpu().numpy()[rows]
    Zref = oracle.aggregate_rows(ref, T, rows)
    bound = oracle.aggregate_rows(ref, np.abs(T), rows)
    err = np.abs(Z.astype(np.float64) - Zref)
    ratio = float((err / (1e-5 * bound + 1e-30)).max())
    print(f"w={w}: max |err|/(1e-5·|Â||T|) = {ratio:.3g} (hubs {float((err[:64] / (1e-5 * bound[:64])).max()):.3g})")
    assert ratio <= 1.0


def test_products_forward_loss(P):
    w = make_workload("products")
    n = w["cfg"].num_nodes
    g, f, m = _model(P, w)
    assert m.order == [1, 0, 0]
    rng = np.random.default_rng(1)
    rows = list(rng.choice(n, 16, replace=False))
    ref_g, rp, ci, dinv = _check_graph(g, w, rows)
    m.forward(1)
    loss = m.loss().item()
    torch.cuda.synchronize()
    ref_loss = _golden_loss1("products")
    assert math.isfinite(loss)
    assert abs(loss - ref_loss) <= 1e-3 * max(1.0, abs(ref_loss)), (loss, ref_loss)
