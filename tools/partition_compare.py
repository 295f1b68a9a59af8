"""Contiguous 1D (north star, D1) vs Alg. 4 Phase III greedy (+ relabelling) partitions, compared on
the quantities of the paper's distributed cost model:

  T_comp ∝ max_r Σ d̃ over rank r's rows (SpMM work)  -> load imbalance max/mean
  T_halo ∝ ghost rows per exchange                   -> total and max ghosts
  cut    = entries of A whose column lives on another rank

Graphs are the bench workloads (synth/) plus a μ (inter-community fraction) sweep on an
arxiv-sized graph.  The CSR is built by the product (mph_graph_build on the GPU) and every
statistic by the product's host code (mph_partition_*), so this needs a GPU box:

    python tools/partition_compare.py [--out profiles/r01_partition_compare.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2512_01678_b200 as P  # noqa: E402
from synth.generate import CONFIGS, make_graph  # noqa: E402


def stats_for(rp, ci, world):
    n = rp.size - 1
    out = {}
    bounds = P.partition_1d(rp, world)
    part_1d = np.repeat(np.arange(world, dtype=np.int32), np.diff(bounds))
    part_g, _ = P.partition_greedy(rp, world)
    for name, part in (("1d", part_1d), ("greedy", part_g)):
        st = P.partition_stats(rp, ci, part, world)
        load = st[:, 1].astype(np.float64)
        out[name] = {"imbalance_max_over_mean": float(load.max() / load.mean()),
                     "ghost_rows_total": int(st[:, 2].sum()), "ghost_rows_max": int(st[:, 2].max()),
                     "cut_fraction": float(st[:, 3].sum() / max(1, rp[-1] - n)),
                     "per_rank": st.tolist()}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/r01_partition_compare.json")
    ap.add_argument("--worlds", default="2,4,8")
    a = ap.parse_args()
    worlds = [int(x) for x in a.worlds.split(",")]
    cases = []
    for name in ("arxiv", "reddit", "products"):
        c = CONFIGS[name]
        cases.append((name, c.num_nodes, c.nnz_a, c.num_classes, c.alpha, c.mu, c.seed))
    ax = CONFIGS["arxiv"]
    for mu in (0.05, 0.2, 0.5):
        cases.append((f"arxiv_mu{mu}", ax.num_nodes, ax.nnz_a, ax.num_classes, ax.alpha, mu, ax.seed))
    res = []
    for (name, n, nnz, c, alpha, mu, seed) in cases:
        t0 = time.time()
        src, dst = make_graph(n, nnz, c, alpha, mu, seed)
        g = P.Graph(src, dst, n)
        rp, ci = (t.cpu().numpy() for t in g.csr()[:2])
        del g
        row = {"graph": name, "nodes": n, "nnz_A": nnz, "mu": mu, "alpha": alpha, "by_world": {}}
        for world in worlds:
            row["by_world"][str(world)] = stats_for(rp, ci, world)
            s = row["by_world"][str(world)]
            print(f"{name:14s} P={world} 1d: imb {s['1d']['imbalance_max_over_mean']:.3f} ghosts {s['1d']['ghost_rows_total']:>9d}"
                  f" cut {s['1d']['cut_fraction']:.3f} | greedy: imb {s['greedy']['imbalance_max_over_mean']:.4f}"
                  f" ghosts {s['greedy']['ghost_rows_total']:>9d} cut {s['greedy']['cut_fraction']:.3f}", flush=True)
        row["seconds"] = time.time() - t0
        res.append(row)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump({"what": "contiguous 1D vs Alg. 4 Phase III greedy + relabel (P:399-492, cost model P:545-569)",
                   "cases": res}, f, indent=1)


if __name__ == "__main__":
    main()
