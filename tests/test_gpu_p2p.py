"""NEXT-1: the NVLink peer-memory halo exchange and fused gradient sum, run as a
real multi-process job on ONE GPU.

Each rank is its own process with its own CUDA context on cuda:0; the ranks map each other's
arenas with CUDA IPC exactly as on an 8-GPU NVSwitch box (same-device IPC mappings take the same
code path: cudaIpcOpenMemHandle, system-scope release/acquire flags, peer loads/stores), and
torch.distributed over gloo only carries the 512-byte arena descriptors (plumbing).  Nothing in
the data path uses NCCL.

Checks, per configuration (dense transform-first, aggregate-first layer 1 whose dinv ⊙ X ghost
rows travel at open, sparse-feature layer 1 with dropout, world 2 and 3):
  * no peer wait timed out (mph_gcn_p2p_status);
  * the replicated parameters and the loss are BITWISE identical on every rank (the fused
    optimizer sums the gradient slabs in rank order on every rank);
  * loss_1..loss_E within 1e-3 of the single-graph FP64 oracle (north star), the first-epoch
    gradient within 2e-3 normwise (reading R1) — distribution transparency;
  * a CUDA-graph-captured P2P epoch replays bitwise equal to eager epochs.
"""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
from synth.generate import make_small

pytestmark = pytest.mark.gpu

CASES = {
    # name: (world, make_small kwargs, dims, force_mode, dropout_p, epochs)
    "dense_tf_w2": (2, dict(n=3000, nnz_a=36000, f=40, c=5, seed=3, alpha=2.1, mu=0.3), (40, 32, 5), 0, 0.0, 6),
    "af_layer1_w3": (3, dict(n=3500, nnz_a=40000, f=24, c=6, seed=4, alpha=2.3, mu=0.4), (24, 64, 48, 6), 0, 0.0, 6),
    "sparse_dropout_w2": (2, dict(n=2500, nnz_a=20000, f=300, c=4, kind="binary", density=0.03, seed=5),
                          (300, 40, 4), 1, 0.25, 6),
    # BF16 GEMM operands: hidden H / backward G stored bf16, the two SpMM parts meet in FP32 scratch
    "bf16_tf_w3": (3, dict(n=3500, nnz_a=40000, f=40, c=5, seed=6, alpha=2.3, mu=0.4), (40, 32, 16, 5), 0, 0.1, 6,
                   "bf16"),
    # SGD with momentum and weight decay through the fused slab-sum optimizer
    "sgd_w2": (2, dict(n=3000, nnz_a=36000, f=40, c=5, seed=7, alpha=2.1, mu=0.3), (40, 32, 5), 0, 0.0, 6, "tf32",
               ("sgd", 0.05, 0.9, 1e-4)),
}


def _case(case):
    c = CASES[case]
    return c[:6] + ((c[6] if len(c) > 6 else "tf32"),)


def _opt(case):
    """(kind, lr, momentum, weight_decay) or None (Adam, the default)."""
    c = CASES[case]
    return c[7] if len(c) > 7 else None


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, result_q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import paper_2512_01678_b200 as P
        _, kw, dims, force_mode, p_drop, epochs, prec = _case(case)
        w = make_small(**kw)
        n = kw["n"]
        gfull = P.Graph(w["src"], w["dst"], n)
        rp, ci = (t.cpu().numpy() for t in gfull.csr()[:2])
        bounds = P.partition_1d(rp, world)
        plan = P.Plan(rp, ci, n, bounds, rank)
        g = P.Graph.from_plan(plan)
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        y = torch.from_numpy(np.ascontiguousarray(w["y"][r0:r1])).cuda()

        def model():
            f = P.Features(torch.from_numpy(np.ascontiguousarray(w["X"][r0:r1])).cuda(), force_mode=force_mode)
            m = P.GCN(g, f, dims, dropout_p=p_drop, dropout_seed=11, comm="p2p", precision=prec)
            m.init_xavier(42)
            m.set_labels(y, n_lab_global=n)
            return f, m

        fa, ma = model()
        losses, grads1 = [], None
        spec = _opt(case)
        cfg = P.optimizer(spec[0], lr=spec[1], momentum=spec[2], weight_decay=spec[3]) if spec else P.api.DEFAULT_ADAM
        for t in range(1, epochs + 1):
            losses.append(ma.train_epoch(t, cfg).item())
            if t == 1:
                grads1 = ma.grads_flat.cpu().numpy().copy()   # the summed gradient of epoch 1
        # the same job as one eager epoch + a captured epoch replayed epochs-1 times
        fb, mb = model()
        replayed = [mb.train_epoch(1, cfg).item()]
        mb.graph_capture(2, cfg)
        for _ in range(epochs - 1):
            replayed.append(mb.replay().item())
        torch.cuda.synchronize()
        res = dict(rank=rank, losses=losses, replayed=replayed, grads1=grads1,
                   params=ma.params_flat.cpu().numpy().copy(), params_b=mb.params_flat.cpu().numpy().copy(),
                   offsets=ma.offsets, ld_w=ma.ld_w, status=(ma.p2p_status(), mb.p2p_status()),
                   order=ma.order, n_ghost=plan.n_ghost)
        dist.barrier()   # nobody unmaps an arena a peer may still read
        del ma, mb
        dist.barrier()
        result_q.put(res)
    except Exception as e:  # pragma: no cover - reported by the parent
        import traceback
        result_q.put(dict(rank=rank, error=f"{e!r}\n{traceback.format_exc()}"))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def _run(case):
    import torch.multiprocessing as mp
    world = CASES[case][0]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    try:
        for _ in range(world):
            r = q.get(timeout=600)
            out[r["rank"]] = r
    finally:
        for p in procs:
            p.join(timeout=120)
            if p.is_alive():
                p.kill()
    errs = [r["error"] for r in out.values() if "error" in r]
    assert not errs, errs[0]
    return [out[r] for r in range(world)]


def _unpack(flat, offsets, ld_w, dims):
    Ws, bs = [], []
    for l in range(len(dims) - 1):
        fin, fout = dims[l], dims[l + 1]
        Ws.append(flat[offsets[2 * l]:offsets[2 * l] + fin * ld_w[l]].reshape(fin, ld_w[l])[:, :fout])
        bs.append(flat[offsets[2 * l + 1]:offsets[2 * l + 1] + fout])
    return Ws, bs


@pytest.mark.parametrize("case", list(CASES))
def test_p2p_epochs_match_oracle(case):
    _check_p2p_case(case)


@pytest.mark.parametrize("case", ["dense_tf_w2", "af_layer1_w3", "bf16_tf_w3"])
def test_p2p_chunked_parts_match_oracle(case, monkeypatch):
    """The owned-edge / ghost-edge launches (parts 0 and 1) over their chunked virtual CSRs
    (MPH_SPMM_SPLIT=2 forces them at this size, chunks of 32 edges), ranks spawned with that
    environment: the same bars as the whole-row-items run."""
    monkeypatch.setenv("MPH_SPMM_SPLIT", "2")
    monkeypatch.setenv("MPH_SPMM_CHUNK_EDGES", "32")
    _check_p2p_case(case)


def _check_p2p_case(case):
    world, kw, dims, force_mode, p_drop, epochs, prec = _case(case)
    res = _run(case)
    for r in res:
        assert r["status"] == (0, 0), f"rank {r['rank']}: a peer-memory wait timed out"
        assert r["n_ghost"] > 0
    if case == "af_layer1_w3":
        assert res[0]["order"][0] == 1   # the Xs setup exchange is exercised
    # replicated state: the same bits on every rank
    for r in res[1:]:
        assert r["losses"] == res[0]["losses"]
        assert np.array_equal(r["params"], res[0]["params"])
        assert np.array_equal(r["grads1"], res[0]["grads1"])
    # CUDA-graph replay of P2P epochs == eager
    for r in res:
        assert r["replayed"] == r["losses"]
        assert np.array_equal(r["params_b"], r["params"])
    # distribution transparency against the single-graph FP64 oracle
    w = make_small(**kw)
    g = oracle.graph_build(w["src"], w["dst"], kw["n"])
    spec = _opt(case)
    okw = dict(optimizer=spec[0], lr=spec[1], momentum=spec[2], weight_decay=spec[3]) if spec else {}
    ref_losses, _ = oracle.train(g, w["X"], w["y"], dims, epochs=epochs, seed=42, dropout_p=p_drop,
                                 dropout_seed=11, **okw)
    got = np.array(res[0]["losses"])
    assert np.all(np.abs(got - ref_losses) <= 1e-3 * np.abs(ref_losses)), (got, ref_losses)
    Ws, bs = oracle.xavier_init(dims, 42)
    Z, cache = oracle.forward(g, w["X"], Ws, bs, p_drop, 11, 1, operand_rounding=None if prec == "tf32" else "bf16")
    _, dZ = oracle.softmax_ce(Z, w["y"])
    dWs, dbs = oracle.backward(g, cache, Ws, dZ)
    gW, gb = _unpack(res[0]["grads1"], res[0]["offsets"], res[0]["ld_w"], dims)
    for l in range(len(dims) - 1):
        for got_g, ref_g in ((gW[l], dWs[l]), (gb[l], dbs[l])):
            rel = np.linalg.norm(got_g - ref_g) / max(np.linalg.norm(ref_g), 1e-30)
            assert rel <= 2e-3, (case, l, rel)


def _worker_fullsize(rank, world, port, rows_per_rank, result_q, config="reddit"):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import paper_2512_01678_b200 as P
        from synth.generate import make_workload
        w = make_workload(config)
        cfg = w["cfg"]
        n = cfg.num_nodes
        gfull = P.Graph(w["src"], w["dst"], n)
        rp, ci = (t.cpu().numpy() for t in gfull.csr()[:2])
        del gfull
        bounds = P.partition_1d(rp, world)
        plan = P.Plan(rp, ci, n, bounds, rank)
        g = P.Graph.from_plan(plan)
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        f = P.Features(torch.from_numpy(np.ascontiguousarray(w["X"][r0:r1])).cuda())
        m = P.GCN(g, f, cfg.dims, comm="p2p")
        m.init_xavier(42)
        m.set_labels(torch.from_numpy(np.ascontiguousarray(w["y"][r0:r1])).cuda(), n_lab_global=n)
        m.forward(1)
        loss1 = m.loss().item()
        rng = np.random.default_rng(rank)
        rows = np.sort(rng.choice(np.arange(r0, r1), rows_per_rank, replace=False))
        H1 = m.tensor(1, 1)[torch.as_tensor(rows - r0, device="cuda")].cpu().numpy()
        m.backward()
        m.adam(1)
        loss2 = m.train_epoch(2).item()
        torch.cuda.synchronize()
        res = dict(rank=rank, loss1=loss1, loss2=loss2, rows=rows, H1=H1, params=m.params_flat.cpu().numpy().copy(),
                   status=m.p2p_status(), n_ghost=plan.n_ghost, bounds=bounds)
        dist.barrier()
        del m
        dist.barrier()
        result_q.put(res)
    except Exception as e:  # pragma: no cover
        import traceback
        result_q.put(dict(rank=rank, error=f"{e!r}\n{traceback.format_exc()}"))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.slow
@pytest.mark.parametrize("config", ["reddit", "products"])
def test_p2p_fullsize_world2(config):
    """BASELINE.json's full-size workloads as 2-rank P2P jobs (each rank half the rows; reddit
    ~120k ghost rows per exchange, products an aggregate-first layer 1 whose dinv ⊙ X ghost rows
    move at open): epoch-1 loss against the FP64 oracle forward, sampled H_1 rows (aggregating
    ghost neighbours) against the oracle within the TF32 bound composed through the aggregation,
    replicas bitwise identical after an optimizer step."""
    import psutil
    if config == "products" and psutil.virtual_memory().available < 64 * 2 ** 30:
        pytest.skip("needs ~64 GB host RAM (two generators + the FP64 oracle at products scale)")
    import torch.multiprocessing as mp
    from synth.generate import make_workload
    world, per = 2, 24
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_fullsize, args=(r, world, port, per, q, config)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    try:
        for _ in range(world):
            r = q.get(timeout=900)
            out[r["rank"]] = r
    finally:
        for p in procs:
            p.join(timeout=120)
            if p.is_alive():
                p.kill()
    errs = [r["error"] for r in out.values() if "error" in r]
    assert not errs, errs[0]
    res = [out[r] for r in range(world)]
    for r in res:
        assert r["status"] == 0 and r["n_ghost"] > 50000
    assert res[0]["loss1"] == res[1]["loss1"] and res[0]["loss2"] == res[1]["loss2"]
    assert np.array_equal(res[0]["params"], res[1]["params"])
    w = make_workload(config)
    cfg = w["cfg"]
    g = oracle.graph_build(w["src"], w["dst"], cfg.num_nodes)
    Ws, bs = oracle.xavier_init(cfg.dims, 42)
    W1 = Ws[0].astype(np.float64)
    d = g.deg.astype(np.float64)
    for r in res:
        lo, hi = int(r["bounds"][r["rank"]]), int(r["bounds"][r["rank"] + 1])
        crossing = 0
        for u, h in zip(r["rows"], r["H1"]):
            nb = g.col_idx[g.row_ptr[u]:g.row_ptr[u + 1]].astype(np.int64)
            crossing += int(np.any((nb < lo) | (nb >= hi)))
            a = 1.0 / np.sqrt(d[u] * d[nb])
            Xn = w["X"][nb].astype(np.float64)
            z = a @ (Xn @ W1)
            lim = 2e-3 * (a @ (np.abs(Xn) @ np.abs(W1))) + 2.0 ** -11 * np.abs(z) + 1e-30
            assert np.all(np.abs(h[:cfg.dims[1]] - np.maximum(z, 0)) <= lim), f"rank {r['rank']} row {u}"
        assert crossing >= len(r["rows"]) // 2   # the sample exercises the pulled ghost rows
    Z, _ = oracle.forward(g, w["X"], Ws, bs)
    ref_loss, _ = oracle.softmax_ce(Z, w["y"])
    assert abs(res[0]["loss1"] - ref_loss) <= 1e-3 * max(1.0, abs(ref_loss)), (res[0]["loss1"], ref_loss)


@pytest.mark.slow
def test_bench_two_ranks_share_device():
    """bench.py's N > 1 code path end to end (torchrun, 2 ranks, P2P transport, max-over-ranks
    timing, e2e) on one GPU via --share-device; the JSON line comes from rank 0."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), os.path.join(root, "bench.py"), "--gpus", "2",
           "--share-device", "--comm", "p2p", "--config", "arxiv", "--steps", "3", "--warmup", "3",
           "--secondary", "none", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["gpu_launches"] > 0
    assert np.isfinite(line["final_loss"]) and line["e2e"]["value"] > 0
    assert "comm p2p" in line["config"]["parallelism"]


def _worker_mismatch(rank, world, port, result_q):
    """Ranks that decide the dense/sparse switch differently must fail loudly at open (advisor
    finding: the rank-local switch gave mismatched exchanges); the global decision agrees."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import paper_2512_01678_b200 as P
        n = 2000
        w = make_small(n, 16000, 16, 4, seed=9)
        X = w["X"].copy()
        gfull = P.Graph(w["src"], w["dst"], n)
        rp, ci = (t.cpu().numpy() for t in gfull.csr()[:2])
        bounds = P.partition_1d(rp, world)
        g = P.Graph.from_plan(P.Plan(rp, ci, n, bounds, rank))
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        if rank == 1:
            X[r0:r1] = 0.0
            X[r0, 0] = 1.0            # rank 1's rows alone are ~100 % sparse, rank 0's dense
        Xd = torch.from_numpy(np.ascontiguousarray(X[r0:r1])).cuda()
        local = P.Features(Xd)         # rank-local switch: rank 0 dense, rank 1 sparse
        mode = P.Features.global_mode(P.Features.count_nnz(Xd), r1 - r0, 16)
        err = ""
        try:
            P.GCN(g, local, (16, 32, 4), comm="p2p", pg=None)   # 16 -> 32: dense gives AF, sparse TF
        except Exception as e:
            err = str(e)
        glob = P.Features(Xd, force_mode=mode)
        m = P.GCN(g, glob, (16, 32, 4), comm="p2p")
        m.init_xavier(42)
        m.set_labels(torch.from_numpy(np.ascontiguousarray(w["y"][r0:r1])).cuda(), n_lab_global=n)
        loss = m.train_epoch(1).item()
        torch.cuda.synchronize()
        res = dict(rank=rank, local_mode=local.mode, mode=mode, err=err, loss=loss, status=m.p2p_status())
        dist.barrier()
        del m
        dist.barrier()
        result_q.put(res)
    except Exception as e:  # pragma: no cover
        import traceback
        result_q.put(dict(rank=rank, error=f"{e!r}\n{traceback.format_exc()}"))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_p2p_mismatched_feature_modes_fail_loudly():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_mismatch, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    try:
        for _ in range(2):
            r = q.get(timeout=300)
            out[r["rank"]] = r
    finally:
        for p in procs:
            p.join(timeout=120)
            if p.is_alive():
                p.kill()
    errs = [r["error"] for r in out.values() if "error" in r]
    assert not errs, errs[0]
    assert [out[r]["local_mode"] for r in (0, 1)] == [0, 1]
    for r in (0, 1):
        assert "feature mode" in out[r]["err"], out[r]["err"]
        assert out[r]["mode"] == out[0]["mode"] == 0
        assert out[r]["status"] == 0
    assert out[0]["loss"] == out[1]["loss"]
