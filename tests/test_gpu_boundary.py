"""The remaining SURVEY §8(b) entry points under their listed names: mph_graph_localize,
mph_halo_plan, mph_gemm (generic shapes), mph_gcn_bind / mph_gcn_workspace_size (caller-owned
state), mph_adam_step and mph_set_allocator (library memory from torch's caching allocator).
Each is checked against the oracle or against the equivalent, already oracle-checked call."""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle
from synth.generate import make_small, make_workload
from tests.gpu_helpers import assert_gemm_close, cuda

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2512_01678_b200 as P
    from paper_2512_01678_b200 import _lib as L
    L.mph_device_check(C.byref(C.c_int32()))
    return P


@pytest.mark.parametrize("world", [2, 3])
def test_graph_localize_and_halo_plan(P, world):
    """mph_graph_localize == plan + graph_from_plan (the oracle-pinned D2-D4 path), bit for bit;
    mph_halo_plan returns the plan's send list / receive slice per peer."""
    n = 2500
    w = make_small(n, 24000, 4, 5, seed=7, alpha=2.2, mu=0.4)
    g = P.Graph(w["src"], w["dst"], n)
    rp, ci = (t.cpu().numpy() for t in g.csr()[:2])
    bounds = P.partition_1d(rp, world)
    for r in range(world):
        lg = g.localize(bounds, r)
        ref = oracle.localize(oracle.graph_build(w["src"], w["dst"], n), bounds, r)
        got_rp, got_ci = (t.cpu().numpy() for t in lg.csr()[:2])
        assert np.array_equal(got_rp, ref.row_ptr) and np.array_equal(got_ci, ref.col_idx)
        plan = P.Plan(rp, ci, n, bounds, r)
        a = plan.arrays()
        for q in range(world):
            h = lg.halo_plan(q)
            s0, s1 = int(a["send_offset"][q]), int(a["send_offset"][q + 1])
            assert np.array_equal(h["send_ids"].cpu().numpy(), a["send_ids"][s0:s1])
            assert h["recv_offset"] == int(a["recv_offset"][q]) and h["n_recv"] == int(a["n_recv"][q])


@pytest.mark.parametrize("M,N,K", [(1000, 48, 104), (3001, 256, 64)])
def test_mph_gemm_generic(P, M, N, K):
    from paper_2512_01678_b200._lib import MorphlingError, mph_gemm
    rng = np.random.default_rng(M)
    A = rng.standard_normal((M, K)).astype(np.float32)
    Bt = rng.standard_normal((N, K)).astype(np.float32)
    s = torch.cuda.current_stream().cuda_stream
    c = torch.zeros((M, N), device="cuda")
    a_d, bt_d = cuda(A), cuda(Bt)   # keep the device inputs alive across the asynchronous call
    mph_gemm(M, N, K, a_d.data_ptr(), K, 0, bt_d.data_ptr(), K, 1, c.data_ptr(), N, 0, 0, s)
    torch.cuda.synchronize()
    assert_gemm_close(c.cpu().numpy(), A, Bt.T, what="mph_gemm NT")
    # transposed-A shape: C[M2, N2] = A2[K2, M2]^T B2[K2, N2] (contraction over K2 = "nodes")
    K2, M2, N2 = 5000, K, N
    A2 = rng.standard_normal((K2, M2)).astype(np.float32)
    B2 = rng.standard_normal((K2, N2)).astype(np.float32)
    c2 = torch.zeros((M2, N2), device="cuda")
    a2_d, b2_d = cuda(A2), cuda(B2)
    mph_gemm(M2, N2, K2, a2_d.data_ptr(), M2, 1, b2_d.data_ptr(), N2, 0, c2.data_ptr(), N2, 0, 0, s)
    torch.cuda.synchronize()
    assert_gemm_close(c2.cpu().numpy(), A2.T, B2, what="mph_gemm TN")
    for bad in ((0, 0, 0), (1, 1, 0), (0, 1, 2)):   # (transA, transB, precision)
        with pytest.raises(MorphlingError) as e:
            mph_gemm(M, N, K, a_d.data_ptr(), K, bad[0], bt_d.data_ptr(), K, bad[1], c.data_ptr(), N, bad[2], 0, s)
        assert e.value.code == -9   # MPH_ENOTSUP


def _model(P, w):
    dims = w["cfg"].dims
    g = P.Graph(w["src"], w["dst"], w["cfg"].num_nodes)
    f = P.Features(cuda(w["X"]))
    m = P.GCN(g, f, dims)
    y = cuda(w["y"].astype(np.int32))
    return g, f, m, y


def test_bind_caller_buffers_and_adam_step(P):
    """Caller-owned params/grads/moments/workspace (torch tensors) give the same epochs, bit for
    bit, as the model's own buffers, and the caller's tensors hold the state; mph_adam_step ==
    mph_gcn_adam."""
    w = make_workload("pubmed")
    _, _, ma, ya = _model(P, w)
    ma.init_xavier(42)
    ma.set_labels(ya)
    ref = [ma.train_epoch(t).item() for t in range(1, 5)]
    _, _, mb, yb = _model(P, w)
    n = mb.num_params
    params, grads = torch.empty(n, device="cuda"), torch.empty(n, device="cuda")
    am, av = torch.empty(n, device="cuda"), torch.empty(n, device="cuda")
    ws = torch.empty(mb.workspace_size(), dtype=torch.uint8, device="cuda")
    mb.bind(params, grads, am, av, ws)
    mb.init_xavier(42)
    mb.set_labels(yb)
    got = []
    for t in range(1, 5):   # forward / loss / backward / mph_adam_step, one call each
        mb.forward(t)
        got.append(mb.loss().item())
        mb.backward()
        from paper_2512_01678_b200._lib import AdamCfg, mph_adam_step
        mph_adam_step(mb.h, C.byref(AdamCfg(0.01, 0.9, 0.999, 1e-8)), t, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert got == ref
    assert torch.equal(params, ma.params_flat) and torch.equal(am, ma.adam_m) and torch.equal(av, ma.adam_v)
    assert mb.params_flat.data_ptr() == params.data_ptr()
    with pytest.raises(Exception):   # a workspace below mph_gcn_workspace_size is refused
        mb.bind(workspace=torch.empty(max(1, mb.workspace_size() // 2), dtype=torch.uint8, device="cuda"))


def test_set_allocator_torch(P):
    """Library memory from torch's caching allocator: same epochs bit for bit, every allocation
    released through the allocator that made it when the handles die."""
    w = make_workload("cora")
    _, _, ma, ya = _model(P, w)
    ma.init_xavier(42)
    ma.set_labels(ya)
    ref = [ma.train_epoch(t).item() for t in range(1, 4)]
    live = P.use_torch_allocator(True)
    try:
        g, f, mb, yb = _model(P, w)
        n_live = len(live)
        assert n_live >= 10   # CSR, features, parameters, activations, workspaces ...
        mb.init_xavier(42)
        mb.set_labels(yb)
        got = [mb.train_epoch(t).item() for t in range(1, 4)]
        assert got == ref
        del mb, f, g
        import gc
        gc.collect()
        torch.cuda.synchronize()
        assert len(live) == 0
    finally:
        P.use_torch_allocator(False)


@pytest.mark.parametrize("M,N,K", [(1000, 48, 104), (3001, 256, 64), (777, 128, 608), (4099, 40, 256)])
def test_mph_gemm_bf16(P, M, N, K):
    """precision 1 (BF16 operands, kind::f16, FP32 accumulate) on both GEMM shapes: against the FP64
    product of the same BF16 values, so only the FP32 accumulation error remains (1e-5 bound)."""
    from paper_2512_01678_b200._lib import mph_gemm
    rng = np.random.default_rng(M + K)
    s = torch.cuda.current_stream().cuda_stream
    ldk = (K + 7) // 8 * 8
    A = torch.zeros((M, ldk), dtype=torch.bfloat16, device="cuda")
    Bt = torch.zeros((N, ldk), dtype=torch.bfloat16, device="cuda")
    A[:, :K] = torch.from_numpy(rng.standard_normal((M, K)).astype(np.float32)).to(torch.bfloat16)
    Bt[:, :K] = torch.from_numpy(rng.standard_normal((N, K)).astype(np.float32)).to(torch.bfloat16)
    c = torch.zeros((M, N), device="cuda")
    mph_gemm(M, N, K, A.data_ptr(), ldk, 0, Bt.data_ptr(), ldk, 1, c.data_ptr(), N, 1, 0, s)
    torch.cuda.synchronize()
    a64, b64 = A[:, :K].double().cpu().numpy(), Bt[:, :K].double().cpu().numpy()
    ref, bound = a64 @ b64.T, np.abs(a64) @ np.abs(b64).T
    assert np.all(np.abs(c.double().cpu().numpy() - ref) <= 1e-5 * bound + 1e-30)
    # transposed-A shape, contraction over K2 "nodes" with MN-major BF16 tiles
    K2, M2, N2 = 7001, (K + 7) // 8 * 8, (N + 7) // 8 * 8
    A2 = torch.from_numpy(rng.standard_normal((K2, M2)).astype(np.float32)).to(torch.bfloat16).cuda()
    B2 = torch.from_numpy(rng.standard_normal((K2, N2)).astype(np.float32)).to(torch.bfloat16).cuda()
    c2 = torch.zeros((M2, N2), device="cuda")
    mph_gemm(M2, N2, K2, A2.data_ptr(), M2, 1, B2.data_ptr(), N2, 0, c2.data_ptr(), N2, 1, 0, s)
    torch.cuda.synchronize()
    a2, b2 = A2.double().cpu().numpy(), B2.double().cpu().numpy()
    ref2, bound2 = a2.T @ b2, np.abs(a2).T @ np.abs(b2)
    assert np.all(np.abs(c2.double().cpu().numpy() - ref2) <= 1e-5 * bound2 + 1e-30)
