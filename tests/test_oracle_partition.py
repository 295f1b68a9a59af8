"""Pins for the oracle's Alg. 4 partitioners (Phase II component bin packing, Phase III
load-aware greedy) and the relabelling that turns a partition
map into contiguous id ranges.  Pinned to hand-worked cases, scipy's connected components, the
list-scheduling bound of the greedy, brute-force recounts, and the permutation invariance of
the whole training step."""
import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.csgraph as csgraph

import oracle
from synth.generate import make_small


def test_greedy_star_hand_case():
    # hub 0 (deg 9) then leaves 1..9 (deg 1); weights add deg + 1:
    # hub -> r0 [10, 0]; leaves 1-5 -> r1 [10, 10]; 6 -> r0 (tie, lower rank) [12, 10];
    # 7 -> r1 [12, 12]; 8 -> r0 [14, 12]; 9 -> r1 [14, 14]
    src = np.zeros(9, np.int32)
    dst = np.arange(1, 10, dtype=np.int32)
    g = oracle.graph_build(src, dst, 10)
    part = oracle.partition_greedy(g, 2)
    assert part.tolist() == [0, 1, 1, 1, 1, 1, 0, 1, 0, 1]
    st = oracle.partition_stats(g, part, 2)
    assert st[:, 1].tolist() == [14, 14]


@pytest.mark.parametrize("seed,world", [(0, 2), (1, 3), (2, 4), (3, 8)])
def test_greedy_list_scheduling_bound(seed, world):
    w = make_small(600, 5000, 4, 3, seed=seed, alpha=2.1)
    g = oracle.graph_build(w["src"], w["dst"], 600)
    part = oracle.partition_greedy(g, world)
    load = np.bincount(part, weights=g.deg.astype(np.float64), minlength=world)
    assert load.sum() == g.deg.sum()
    # the greedy puts every node on the least-loaded rank, so max - min <= the largest item
    assert load.max() - load.min() <= g.deg.max()


def test_components_hand_case_and_ties():
    # components {0..4} (path), {5,6,7} (triangle), {8,9}, {10,11}; world 2:
    # sizes 5, 3, 2, 2: 5 -> r0 [5, 0]; 3 -> r1 [5, 3]; {8, 9} -> r1 (3 < 5) [5, 5];
    # {10, 11} -> tie, lower rank -> r0 [7, 5]
    src = np.array([0, 1, 2, 3, 5, 6, 7, 8, 10], np.int32)
    dst = np.array([1, 2, 3, 4, 6, 7, 5, 9, 11], np.int32)
    g = oracle.graph_build(src, dst, 12)
    part, nc = oracle.partition_components(g, 2)
    assert nc == 4
    assert part.tolist() == [0] * 5 + [1] * 3 + [1, 1] + [0, 0]
    # reading R10: loads [7, 5] exceed 1.05 x the mean 6 -> Phase III
    h, phase = oracle.partition_hierarchical(g, 2)
    assert phase == 3 and np.array_equal(h, oracle.partition_greedy(g, 2))
    # without {10, 11}: sizes 5, 3, 2 -> [5, 5], balanced -> Phase II keeps the packing
    g10 = oracle.graph_build(src[:-1], dst[:-1], 10)
    part10, _ = oracle.partition_components(g10, 2)
    h, phase = oracle.partition_hierarchical(g10, 2)
    assert phase == 2 and np.array_equal(h, part10) and part10.tolist() == [0] * 5 + [1] * 5


def test_hierarchical_giant_component_and_too_few_components_fall_through():
    # a giant path 0..19 plus isolated nodes 20, 21: Phase II would put 20 of 22 nodes on one rank
    src = np.arange(0, 19, dtype=np.int32)
    g = oracle.graph_build(src, src + 1, 22)
    assert oracle.connected_components(g)[1] == 3
    part, phase = oracle.partition_hierarchical(g, 2)
    assert phase == 3 and np.array_equal(part, oracle.partition_greedy(g, 2))
    # two equal components but four ranks: two bins would stay empty
    s2 = np.array([0, 1, 2, 4, 5, 6], np.int32)
    g2 = oracle.graph_build(s2, s2 + 1, 8)
    part, phase = oracle.partition_hierarchical(g2, 4)
    assert phase == 3
    part, phase = oracle.partition_hierarchical(g2, 2)
    assert phase == 2 and part.tolist() == [0] * 4 + [1] * 4


def test_components_match_scipy_and_connected_fallthrough():
    w = make_small(400, 300, 4, 3, seed=5)                   # sparse enough to be disconnected
    g = oracle.graph_build(w["src"], w["dst"], 400)
    comp, nc = oracle.connected_components(g)
    A = sp.csr_matrix((np.ones(g.nnz), g.col_idx, g.row_ptr), shape=(400, 400))
    nc2, lab = csgraph.connected_components(A, directed=False)
    assert nc == nc2 > 1
    # same partition of the nodes (labels may be numbered differently)
    pairs = set(zip(comp.tolist(), lab.tolist()))
    assert len(pairs) == nc
    # a connected graph falls through to Phase III
    wc = make_small(200, 3000, 4, 3, seed=6)
    gc = oracle.graph_build(wc["src"], wc["dst"], 200)
    assert oracle.connected_components(gc)[1] == 1
    part, phase = oracle.partition_hierarchical(gc, 3)
    assert phase == 3 and np.array_equal(part, oracle.partition_greedy(gc, 3))


def test_relabel_is_contiguous_and_order_preserving():
    rng = np.random.default_rng(0)
    part = rng.integers(0, 4, 1000).astype(np.int32)
    new_id, bounds = oracle.relabel(part, 4)
    assert sorted(new_id.tolist()) == list(range(1000))                  # a bijection
    for r in range(4):
        olds = np.nonzero(part == r)[0]                                   # ascending old ids
        assert new_id[olds].tolist() == list(range(bounds[r], bounds[r + 1]))


def test_partition_stats_brute_force():
    w = make_small(150, 900, 4, 3, seed=8)
    g = oracle.graph_build(w["src"], w["dst"], 150)
    part = oracle.partition_greedy(g, 3)
    st = oracle.partition_stats(g, part, 3)
    nb = [set() for _ in range(150)]
    for a, b in zip(w["src"].tolist(), w["dst"].tolist()):
        if a != b:
            nb[a].add(b)
            nb[b].add(a)
    for r in range(3):
        own = [v for v in range(150) if part[v] == r]
        ghosts = {u for v in own for u in nb[v] if part[u] != r}
        cut = sum(1 for v in own for u in nb[v] if part[u] != r)
        assert st[r].tolist() == [len(own), sum(len(nb[v]) + 1 for v in own), len(ghosts), cut]


def test_training_is_invariant_under_relabelling():
    """The loss is a mean over nodes and Ã is relabelled with its rows and columns, so training on
    the relabelled graph with permuted features and labels gives the same trajectory."""
    n = 300
    w = make_small(n, 2500, 6, 3, seed=9)
    g = oracle.graph_build(w["src"], w["dst"], n)
    part = oracle.partition_greedy(g, 3)
    new_id, _ = oracle.relabel(part, 3)
    g2 = oracle.graph_build(new_id[w["src"]].astype(np.int32), new_id[w["dst"]].astype(np.int32), n)
    inv = np.empty(n, dtype=np.int64)
    inv[new_id] = np.arange(n)
    l1, p1 = oracle.train(g, w["X"], w["y"], (6, 8, 3), epochs=4, seed=42)
    l2, p2 = oracle.train(g2, w["X"][inv], w["y"][inv], (6, 8, 3), epochs=4, seed=42)
    assert np.allclose(l1, l2, rtol=1e-12)
    assert all(np.allclose(a, b, rtol=1e-10, atol=1e-14) for a, b in zip(p1, p2))
