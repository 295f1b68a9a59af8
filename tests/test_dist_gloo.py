"""World-size-2/3 CPU tests (gloo) of the distributed host logic (a10/a11).

Each rank builds its plan with the PRODUCT's host code (mph_partition_1d, mph_plan_create),
then exchanges halo rows over gloo exactly as the plan prescribes (send lists -> ghost slices,
P:517-523) and all-reduces gradients.  The FP64 arithmetic on each rank is the
oracle's definition restricted to the local view.  Checks: halo symmetry across ranks, ghost
rows bit-equal their owners' rows after the exchange, and the summed per-rank loss and
gradients equal the single-graph oracle (distribution transparency).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from synth.generate import make_small


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _exchange(plan_arrays, n_own, buf, rank, world):
    """Halo exchange of rows of `buf` [n_own + n_ghost, w] following the plan (gloo p2p)."""
    reqs = []
    recv_bufs = {}
    for q in range(world):
        if q == rank:
            continue
        s0, s1 = plan_arrays["send_offset"][q], plan_arrays["send_offset"][q + 1]
        if s1 > s0:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(buf[plan_arrays["send_ids"][s0:s1]])), q))
        nr = int(plan_arrays["n_recv"][q])
        if nr:
            t = torch.empty((nr, buf.shape[1]), dtype=torch.float64)
            recv_bufs[q] = t
            reqs.append(dist.irecv(t, q))
    for r in reqs:
        r.wait()
    for q, t in recv_bufs.items():
        o = n_own + int(plan_arrays["recv_offset"][q])
        buf[o:o + t.shape[0]] = t.numpy()


def _local_agg(a, n_own, buf):
    d = a["deg_local"].astype(np.float64)
    out = np.zeros((n_own, buf.shape[1]))
    for i in range(n_own):
        cols = a["col_idx"][a["row_ptr"][i]:a["row_ptr"][i + 1]]
        out[i] = (1.0 / np.sqrt(d[i] * d[cols])) @ buf[cols]
    return out


def _worker(rank, world, port, n, m, result_q, partition="1d"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_01678_b200 import Plan, partition_1d, partition_greedy, relabel
        w = make_small(n, m, 5, 3, seed=17, alpha=2.1, mu=0.3)
        g0 = oracle.graph_build(w["src"], w["dst"], n)
        X0, y0 = w["X"], w["y"]
        if partition == "greedy":
            # Alg. 4 Phase III, then relabel so each rank's nodes are one contiguous range (NEXT-3)
            new_id, bounds = relabel(partition_greedy(g0.row_ptr, world)[0], world)
            inv = np.empty(n, dtype=np.int64)
            inv[new_id] = np.arange(n)
            g = oracle.graph_build(new_id[w["src"]].astype(np.int32), new_id[w["dst"]].astype(np.int32), n)
            w = dict(w, X=X0[inv], y=y0[inv])
        else:
            g = g0
            bounds = partition_1d(g.row_ptr, world)
        plan = Plan(g.row_ptr, g.col_idx, n, bounds, rank)
        a = plan.arrays()
        n_own, row0 = plan.n_own, plan.row0
        gl = np.concatenate([np.arange(row0, row0 + n_own), a["ghosts"]])

        # halo symmetry: what I send to q is exactly q's ghost slice for me
        sent = [None] * world
        mine = {q: (row0 + a["send_ids"][a["send_offset"][q]:a["send_offset"][q + 1]]).tolist() for q in range(world)}
        dist.all_gather_object(sent, mine)
        for q in range(world):
            if q == rank:
                continue
            o, k = int(a["recv_offset"][q]), int(a["n_recv"][q])
            assert sent[q][rank] == a["ghosts"][o:o + k].tolist()

        dims = (5, 8, 3)
        Ws, bs = oracle.xavier_init(dims, 42)
        X = w["X"].astype(np.float64)
        # forward: T = H W on owned rows, exchange ghost rows, aggregate, ...
        H_own = X[row0:row0 + n_own]
        Hs, Zs = [H_own], []
        for l in range(2):
            buf = np.zeros((len(gl), dims[l + 1]))
            buf[:n_own] = Hs[-1] @ Ws[l]
            _exchange(a, n_own, buf, rank, world)
            full_T = X @ Ws[0] if l == 0 else None
            if full_T is not None:                      # ghosts bit-equal the owners' rows
                assert np.array_equal(buf[n_own:], full_T[a["ghosts"]])
            Z = _local_agg(a, n_own, buf) + bs[l]
            Zs.append(Z)
            Hs.append(np.maximum(Z, 0) if l == 0 else Z)
        loss, dZ = oracle.softmax_ce(Zs[1], w["y"][row0:row0 + n_own], n_lab=n)   # global N
        grads = []
        for l in (1, 0):
            buf = np.zeros((len(gl), dims[l + 1]))
            buf[:n_own] = dZ
            _exchange(a, n_own, buf, rank, world)
            G = _local_agg(a, n_own, buf)
            grads = [Hs[l].T @ G, dZ.sum(0)] + grads
            if l == 1:
                dZ = (G @ Ws[1].T) * (Zs[0] > 0)
        flat = torch.from_numpy(np.concatenate([x.ravel() for x in grads] + [np.array([loss])]))
        dist.all_reduce(flat)                           # a11
        if rank == 0:   # the single-graph oracle on the ORIGINAL ids (relabelling must not matter)
            Z, cache = oracle.forward(g0, X0.astype(np.float64), Ws, bs)
            lref, dZr = oracle.softmax_ce(Z, y0)
            dWs, dbs = oracle.backward(g0, cache, Ws, dZr)
            ref = np.concatenate([dWs[0].ravel(), dbs[0], dWs[1].ravel(), dbs[1], [lref]])
            result_q.put(float(np.max(np.abs(flat.numpy() - ref) / (np.abs(ref) + 1e-12))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,partition", [(2, "1d"), (3, "1d"), (2, "greedy"), (3, "greedy")])
def test_distributed_epoch_over_gloo(world, partition):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 240, 1800, q, partition)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    rel = q.get(timeout=5)
    assert rel < 1e-10, rel
