"""Pins for the oracle's distributed plans (c.2 D1-D5).

References: brute-force recounts written here, the union / symmetry invariants
of S:613-615 and S:593, and distribution transparency: the
sum over ranks of per-rank losses and gradients, computed on the local views
with ghost rows filled from their owners, equals the single-graph oracle.
"""
import numpy as np
import pytest

import oracle
from synth.generate import make_small


def _graph(n=400, m=3000, seed=3, alpha=2.1):
    w = make_small(n, m, 6, 4, seed=seed, alpha=alpha)
    return w, oracle.graph_build(w["src"], w["dst"], n)


def test_partition_world1_and_balance():
    _, g = _graph()
    assert oracle.partition_1d(g.row_ptr, 1).tolist() == [0, g.num_nodes]
    for world in (2, 3, 4, 8):
        b = oracle.partition_1d(g.row_ptr, world)
        assert b[0] == 0 and b[-1] == g.num_nodes and np.all(np.diff(b) >= 0)
        # brute force of D1: smallest u with world*row_ptr[u] >= r*nnz
        for r in range(world + 1):
            cand = [u for u in range(g.num_nodes + 1) if world * g.row_ptr[u] >= r * g.nnz]
            assert b[r] == cand[0]
        loads = np.diff(g.row_ptr[b])
        assert loads.max() - g.nnz / world <= g.deg.max()          # within one row of the ideal


@pytest.mark.parametrize("world", [2, 3, 4])
def test_localize_invariants(world):
    _, g = _graph()
    b = oracle.partition_1d(g.row_ptr, world)
    plans = [oracle.localize(g, b, r) for r in range(world)]
    union = set()
    for p in plans:
        gl = np.concatenate([np.arange(p.row0, p.row0 + p.n_own), p.ghosts])
        # brute-force ghost recount
        expect = set()
        for u in range(p.row0, p.row0 + p.n_own):
            for v in g.col_idx[g.row_ptr[u]:g.row_ptr[u + 1]]:
                if not (p.row0 <= v < p.row0 + p.n_own):
                    expect.add(int(v))
        assert sorted(expect) == p.ghosts.tolist()
        for i in range(p.n_own):
            row = p.col_idx[p.row_ptr[i]:p.row_ptr[i + 1]]
            assert np.all(np.diff(row) > 0)
            assert np.all(row[:p.split[i]] < p.n_own) and np.all(row[p.split[i]:] >= p.n_own)
            for c in row:
                union.add((p.row0 + i, int(gl[c])))
    assert union == set(zip(g.rows.tolist(), g.col_idx.tolist()))         # union = global set
    for r in range(world):                                                 # halo symmetry
        for q in range(world):
            if q == r:
                continue
            sent = plans[r].send_ids[q] + plans[r].row0
            o, n = plans[q].recv_offset[r], plans[q].n_recv[r]
            assert np.array_equal(sent, plans[q].ghosts[o:o + n])


def test_distribution_transparency():
    """Per-rank forward/backward over local views (+ ghost rows copied from owners)
    sums to the single-graph oracle (D5)."""
    w, g = _graph(n=300, m=2400, seed=9)
    dims = (6, 8, 4)
    Ws, bs = oracle.xavier_init(dims, 42)
    X = w["X"].astype(np.float64)
    Z, cache = oracle.forward(g, X, Ws, bs)
    loss, dZ = oracle.softmax_ce(Z, w["y"])
    dWs, dbs = oracle.backward(g, cache, Ws, dZ)

    world = 3
    bnd = oracle.partition_1d(g.row_ptr, world)
    plans = [oracle.localize(g, bnd, r) for r in range(world)]
    d = g.deg.astype(np.float64)

    def local_agg(p, full):  # rows of Â·full for owned nodes using only [own | ghosts] rows
        gl = np.concatenate([np.arange(p.row0, p.row0 + p.n_own), p.ghosts])
        vals = full[gl]                                                    # "after the exchange"
        out = np.zeros((p.n_own, full.shape[1]))
        for i in range(p.n_own):
            cols = p.col_idx[p.row_ptr[i]:p.row_ptr[i + 1]]
            out[i] = (1.0 / np.sqrt(d[p.row0 + i] * d[gl[cols]])) @ vals[cols]
        return out

    # forward layer by layer, exchanging the transform output each layer
    H = X
    hs = [X]
    zs = []
    for l in range(2):
        P = H @ Ws[l]
        Zl = np.concatenate([local_agg(p, P) for p in plans]) + bs[l]
        zs.append(Zl)
        H = np.maximum(Zl, 0) if l == 0 else Zl
        hs.append(H)
    total_loss = 0.0
    dz_parts = []
    for p in plans:
        sl = slice(p.row0, p.row0 + p.n_own)
        li, dzi = oracle.softmax_ce(zs[1][sl], w["y"][sl], n_lab=g.num_nodes)   # global N
        total_loss += li
        dz_parts.append(dzi)
    assert abs(total_loss - loss) <= 1e-12 * abs(loss)
    dZ2 = np.concatenate(dz_parts)
    G2 = np.concatenate([local_agg(p, dZ2) for p in plans])
    dW2 = sum(hs[1][p.row0:p.row0 + p.n_own].T @ G2[p.row0:p.row0 + p.n_own] for p in plans)
    assert np.allclose(dW2, dWs[1], rtol=1e-12, atol=1e-15)
    dZ1 = (G2 @ Ws[1].T) * (zs[0] > 0)
    G1 = np.concatenate([local_agg(p, dZ1) for p in plans])
    dW1 = sum(X[p.row0:p.row0 + p.n_own].T @ G1[p.row0:p.row0 + p.n_own] for p in plans)
    db1 = sum(dZ1[p.row0:p.row0 + p.n_own].sum(0) for p in plans)
    assert np.allclose(dW1, dWs[0], rtol=1e-12, atol=1e-15)
    assert np.allclose(db1, dbs[0], rtol=1e-12, atol=1e-15)
