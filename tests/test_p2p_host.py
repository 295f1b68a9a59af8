"""NEXT-1 host-side invariant (CPU): the peer-memory halo PULLS ghost row j of owner q from q's
buffer at local row ghosts[j] - row0_q (p2p.cu, p2p_open), while the NCCL path PUSHES q's send
list to the same ghost slots.  Both address the same rows in the same order iff the
plan's send list of q towards r equals r's ghosts owned by q minus row0_q — checked here with the
product's own plans at several world sizes, and against the oracle's D3/D4 lists."""
import numpy as np
import pytest

import oracle
from synth.generate import make_small


@pytest.mark.parametrize("world", [2, 3, 5, 8])
def test_pull_addressing_equals_send_lists(world):
    from paper_2512_01678_b200 import Plan, partition_1d
    n = 1500
    w = make_small(n, 16000, 4, 5, seed=world, alpha=2.2, mu=0.4)
    g = oracle.graph_build(w["src"], w["dst"], n)
    bounds = partition_1d(g.row_ptr, world)
    plans = [Plan(g.row_ptr, g.col_idx, n, bounds, r) for r in range(world)]
    arrs = [p.arrays() for p in plans]
    for r in range(world):
        a = arrs[r]
        ghosts = a["ghosts"]
        assert np.all(np.diff(ghosts) > 0)  # grouped by owner, ascending (D4)
        for q in range(world):
            o, k = int(a["recv_offset"][q]), int(a["n_recv"][q])
            mine = ghosts[o:o + k]
            assert np.all((mine >= bounds[q]) & (mine < bounds[q + 1]))
            pull_rows = mine - bounds[q]
            s0, s1 = int(arrs[q]["send_offset"][r]), int(arrs[q]["send_offset"][r + 1])
            assert np.array_equal(pull_rows, arrs[q]["send_ids"][s0:s1])
            assert pull_rows.size == 0 or pull_rows.max() < (1 << 27)  # fits the ghost_ref packing
        ref = oracle.localize(g, bounds, r)
        assert np.array_equal(ghosts, ref.ghosts)
