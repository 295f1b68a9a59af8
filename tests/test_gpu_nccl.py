"""a10/a11 over NCCL at world 2 (pack + grouped ncclSend/ncclRecv into the ghost
rows, ncclAllReduce of [dW, db] and the loss), one process per GPU.

NCCL refuses two ranks on one device, so this needs >= 2 visible GPUs and skips otherwise (the
peer-memory transport is exercised on one GPU by test_gpu_p2p.py).  Checks, like the P2P test:
losses and replicated parameters bitwise identical on both ranks, loss_1..loss_6 within 1e-3 of
the single-graph FP64 oracle, first-epoch gradients within 2e-3 normwise (reading R1), the dense
transform-first, aggregate-first-layer-1 and global-switch cases."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
from synth.generate import make_small

pytestmark = pytest.mark.gpu

CASES = {
    "dense_tf": (dict(n=3000, nnz_a=36000, f=40, c=5, seed=3, alpha=2.1, mu=0.3), (40, 32, 5)),
    "af_layer1": (dict(n=3500, nnz_a=40000, f=24, c=6, seed=4, alpha=2.3, mu=0.4), (24, 64, 48, 6)),
}
EPOCHS = 6


def _needs_two_gpus():
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("NCCL transport needs >= 2 GPUs (one rank per device)")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
        import paper_2512_01678_b200 as P
        kw, dims = CASES[case]
        w = make_small(**kw)
        n = kw["n"]
        gfull = P.Graph(w["src"], w["dst"], n)
        rp, ci = (t.cpu().numpy() for t in gfull.csr()[:2])
        bounds = P.partition_1d(rp, world)
        plan = P.Plan(rp, ci, n, bounds, rank)
        g = P.Graph.from_plan(plan)
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        Xd = torch.from_numpy(np.ascontiguousarray(w["X"][r0:r1])).cuda()
        mode = P.Features.global_mode(P.Features.count_nnz(Xd), r1 - r0, kw["f"])
        f = P.Features(Xd, force_mode=mode)
        comm = P.Comm(world, rank)
        m = P.GCN(g, f, dims, comm=comm)
        m.init_xavier(42)
        m.set_labels(torch.from_numpy(np.ascontiguousarray(w["y"][r0:r1])).cuda())   # n_lab summed over ranks
        losses, grads1 = [], None
        for t in range(1, EPOCHS + 1):
            losses.append(m.train_epoch(t).item())
            if t == 1:
                grads1 = m.grads_flat.cpu().numpy().copy()
        torch.cuda.synchronize()
        q.put(dict(rank=rank, losses=losses, grads1=grads1, params=m.params_flat.cpu().numpy().copy(),
                   offsets=m.offsets, ld_w=m.ld_w, order=m.order, n_ghost=plan.n_ghost))
        dist.barrier()
    except Exception as e:  # pragma: no cover
        import traceback
        q.put(dict(rank=rank, error=f"{e!r}\n{traceback.format_exc()}"))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def _unpack(flat, offsets, ld_w, dims):
    Ws, bs = [], []
    for l in range(len(dims) - 1):
        fin, fout = dims[l], dims[l + 1]
        Ws.append(flat[offsets[2 * l]:offsets[2 * l] + fin * ld_w[l]].reshape(fin, ld_w[l])[:, :fout])
        bs.append(flat[offsets[2 * l + 1]:offsets[2 * l + 1] + fout])
    return Ws, bs


@pytest.mark.parametrize("case", list(CASES))
def test_nccl_world2_matches_oracle(case):
    _needs_two_gpus()
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    try:
        for _ in range(2):
            r = q.get(timeout=600)
            out[r["rank"]] = r
    finally:
        for p in procs:
            p.join(timeout=120)
            if p.is_alive():
                p.kill()
    errs = [r["error"] for r in out.values() if "error" in r]
    assert not errs, errs[0]
    a, b = out[0], out[1]
    assert a["n_ghost"] > 0 and b["n_ghost"] > 0
    assert a["losses"] == b["losses"]                       # the all-reduced loss is the same number
    assert np.array_equal(a["params"], b["params"])        # replicated Adam on all-reduced gradients
    kw, dims = CASES[case]
    if case == "af_layer1":
        assert a["order"][0] == 1
    w = make_small(**kw)
    g = oracle.graph_build(w["src"], w["dst"], kw["n"])
    ref, _ = oracle.train(g, w["X"], w["y"], dims, epochs=EPOCHS, seed=42)
    got = np.array(a["losses"])
    assert np.all(np.abs(got - ref) <= 1e-3 * np.maximum(1.0, np.abs(ref))), (got, ref)
    Ws, bs = oracle.xavier_init(dims, 42)
    Z, cache = oracle.forward(g, w["X"], Ws, bs)
    _, dZ = oracle.softmax_ce(Z, w["y"])
    dWs, dbs = oracle.backward(g, cache, Ws, dZ)
    gW, gb = _unpack(a["grads1"], a["offsets"], a["ld_w"], dims)
    for l in range(len(dims) - 1):
        for got_g, ref_g in ((gW[l], dWs[l]), (gb[l], dbs[l])):
            rel = np.linalg.norm(got_g - ref_g) / max(np.linalg.norm(ref_g), 1e-30)
            assert rel <= 2e-3, (case, l, rel)
