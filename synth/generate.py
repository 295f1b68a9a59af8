"""Deterministic synthetic GCN workloads shaped like the paper's datasets.

Recipe: SURVEY.md §8(d) d.1 (degree-corrected planted partition, Chung–Lu
style), restated in DESIGN.md §"Input recipe".  The paper gives no degree or
locality parameters; alpha/mu below are the stated assumptions of d.1.

Shapes (BASELINE.json `configs`; dataset table PAPER.md P:623-644 for Reddit,
ogbn-arxiv and ogbn-products; Cora/Pubmed come from BASELINE.json only):

  cora      2,708 nodes      10,556 nnz(A)  1433-16-7       binary 1.27 %
  pubmed   19,717 nodes      88,648 nnz(A)   500-64-3       tf-idf 10 %
  arxiv   169,343 nodes   1,166,242 nnz(A)   128-256-256-40 dense
  reddit  232,965 nodes 114,615,892 nnz(A)   602-128-41     dense
  products 2,449,029 nodes 61,859,140 nnz(A) 100-256-256-47 dense

`nnz(A)` counts directed entries of the symmetric 0/1 adjacency without
self-loops, so the generator emits exactly nnz(A)/2 undirected
pairs.  All randomness comes from numpy's PCG64 seeded per config, plus a
splitmix64 hash for the exact-count selection, so every call regenerates the
same arrays bit for bit.

This module holds no arithmetic of the method itself.
"""
from __future__ import annotations

import dataclasses
import numpy as np
import torch  # used only for its multithreaded, deterministic searchsorted


def _searchsorted(cdf: np.ndarray, q: np.ndarray) -> np.ndarray:
    return torch.searchsorted(torch.from_numpy(cdf), torch.from_numpy(q), right=True).numpy()


def _sorted_unique(a: np.ndarray) -> np.ndarray:
    a = np.sort(a)
    if a.size == 0:
        return a
    keep = np.empty(a.size, dtype=bool)
    keep[0] = True
    np.not_equal(a[1:], a[:-1], out=keep[1:])
    return a[keep]

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)


@dataclasses.dataclass(frozen=True)
class WorkloadConfig:
    name: str
    num_nodes: int
    nnz_a: int            # directed entries of A (no self loops); pairs = nnz_a // 2
    dims: tuple           # (F, hidden..., C)
    feature_kind: str     # "dense" | "binary" | "tfidf"
    density: float        # target nnz(X)/(N*F) for sparse kinds
    alpha: float          # power-law exponent of expected degrees
    mu: float             # fraction of inter-community edges
    seed: int

    @property
    def num_features(self) -> int:
        return self.dims[0]

    @property
    def num_classes(self) -> int:
        return self.dims[-1]

    @property
    def num_layers(self) -> int:
        return len(self.dims) - 1


CONFIGS = {
    "cora": WorkloadConfig("cora", 2708, 10556, (1433, 16, 7), "binary", 0.0127, 2.5, 0.19, 1),
    "pubmed": WorkloadConfig("pubmed", 19717, 88648, (500, 64, 3), "tfidf", 0.10, 2.5, 0.20, 2),
    "arxiv": WorkloadConfig("arxiv", 169343, 1166242, (128, 256, 256, 40), "dense", 1.0, 2.5, 0.35, 3),
    "reddit": WorkloadConfig("reddit", 232965, 114615892, (602, 128, 41), "dense", 1.0, 2.1, 0.24, 4),
    "products": WorkloadConfig("products", 2449029, 61859140, (100, 256, 256, 47), "dense", 1.0, 2.1, 0.19, 5),
}


def _splitmix64_mix(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    z = x.astype(np.uint64, copy=True)
    z += _GOLDEN
    z ^= z >> np.uint64(30)
    z *= np.uint64(0xBF58476D1CE4E5B9)
    z ^= z >> np.uint64(27)
    z *= np.uint64(0x94D049BB133111EB)
    z ^= z >> np.uint64(31)
    return z


def _blocks(n: int, c: int):
    """C contiguous id blocks, the first n % c get one extra node."""
    base, extra = divmod(n, c)
    sizes = np.full(c, base, dtype=np.int64)
    sizes[:extra] += 1
    starts = np.zeros(c + 1, dtype=np.int64)
    np.cumsum(sizes, out=starts[1:])
    return starts


def make_labels(n: int, c: int) -> np.ndarray:
    starts = _blocks(n, c)
    y = np.zeros(n, dtype=np.int32)
    for b in range(c):
        y[starts[b]:starts[b + 1]] = b
    return y


def make_graph(n: int, nnz_a: int, c: int, alpha: float, mu: float, seed: int):
    """Return (src, dst) int32 arrays with exactly nnz_a // 2 distinct undirected pairs.

    No self loops, no duplicate pairs; direction of each pair is randomised so
    the consumer's symmetrisation is exercised.
    """
    if n <= 1 or nnz_a <= 0:
        return np.zeros(0, np.int32), np.zeros(0, np.int32)
    m = nnz_a // 2
    max_pairs = n * (n - 1) // 2
    if m > max_pairs:
        raise ValueError("too many edges for node count")
    rng = np.random.Generator(np.random.PCG64(seed))
    starts = _blocks(n, c)
    block_of = np.repeat(np.arange(c, dtype=np.int64), np.diff(starts))
    perm = rng.permutation(n)
    w = (perm.astype(np.float64) + 1.0) ** (-1.0 / (alpha - 1.0))
    w *= nnz_a / w.sum()
    np.minimum(w, np.sqrt(w.sum()), out=w)
    cdf = np.cumsum(w)
    total = cdf[-1]
    cdf_lo = np.concatenate([[0.0], cdf])[starts[:-1]]
    cdf_hi = cdf[starts[1:] - 1]

    keys = np.zeros(0, dtype=np.int64)
    draw = int(m * 1.15) + 1024
    for _ in range(64):
        r = rng.random(draw) * total
        u = _searchsorted(cdf, r)
        np.minimum(u, n - 1, out=u)
        local = rng.random(draw) >= mu
        r2 = rng.random(draw)
        bu = block_of[u]
        lo, hi = cdf_lo[bu], cdf_hi[bu]
        r_local = lo + r2 * (hi - lo)
        r_glob = r2 * total
        v = _searchsorted(cdf, np.where(local, r_local, r_glob))
        np.minimum(v, n - 1, out=v)
        ok = u != v
        a = np.minimum(u[ok], v[ok]).astype(np.int64)
        b = np.maximum(u[ok], v[ok]).astype(np.int64)
        keys = _sorted_unique(np.concatenate([keys, a * n + b]))
        if keys.size >= m:
            break
        missing = m - keys.size
        draw = int(missing * 2.0) + 1024
        if draw > 50 * m + 1024:
            draw = 50 * m + 1024
    if keys.size < m:
        # dense fallback for tiny graphs: take pairs uniformly
        all_a, all_b = np.triu_indices(n, 1)
        extra = np.setdiff1d(all_a.astype(np.int64) * n + all_b, keys)
        keys = _sorted_unique(np.concatenate([keys, extra]))
    if keys.size > m:
        h = _splitmix64_mix(keys.astype(np.uint64) ^ np.uint64(seed))
        keep = np.argpartition(h, m - 1)[:m]
        keys = np.sort(keys[keep])
    src = (keys // n).astype(np.int32)
    dst = (keys % n).astype(np.int32)
    flip = (_splitmix64_mix(keys.astype(np.uint64) + np.uint64(seed)) & np.uint64(1)).astype(bool)
    src[flip], dst[flip] = dst[flip].copy(), src[flip].copy()
    order = rng.permutation(m)
    return src[order].copy(), dst[order].copy()


def make_features(n: int, f: int, y: np.ndarray, c: int, kind: str, density: float, seed: int) -> np.ndarray:
    """f32 [n, f] features; every value exactly representable (dyadic)."""
    rng = np.random.Generator(np.random.PCG64(seed + 7919))
    if kind == "dense":
        sigma = np.where(rng.random((c, f)) < 0.5, -1.0, 1.0).astype(np.float32)
        x = np.empty((n, f), dtype=np.float32)
        chunk = max(1, (1 << 24) // max(f, 1))
        for s in range(0, n, chunk):
            e = min(n, s + chunk)
            q = (rng.integers(0, 1 << 21, size=(e - s, f)) - (1 << 20)).astype(np.float32) * np.float32(2.0 ** -20)
            x[s:e] = q + np.float32(0.5) * sigma[y[s:e]]
        return x
    if kind not in ("binary", "tfidf"):
        raise ValueError(kind)
    p_hi = max(0.05, 2.0 * density)
    p_lo = max(0.0, (density - p_hi / c) / (1.0 - 1.0 / c))
    k = np.arange(f)
    hot = (k[None, :] % c) == y[:, None]
    p = np.where(hot, p_hi, p_lo)
    mask = rng.random((n, f)) < p
    if kind == "binary":
        return mask.astype(np.float32)
    vals = rng.integers(1, (1 << 20) + 1, size=(n, f)).astype(np.float32) * np.float32(2.0 ** -22)
    return np.where(mask, vals, np.float32(0.0)).astype(np.float32)


def make_features_csr(n: int, f: int, y: np.ndarray, c: int, density: float, seed: int):
    """Binary sparse features generated directly in CSR form (same mask recipe as
    make_features, for shapes whose dense matrix would not fit host memory, e.g. NELL's
    65,755 x 61,278).  Returns (ptr int64[n+1], idx int32 ascending per row, val f32 == 1)."""
    rng = np.random.Generator(np.random.PCG64(seed + 7919))
    p_hi = max(0.05, 2.0 * density)
    p_lo = max(0.0, (density - p_hi / c) / (1.0 - 1.0 / c))
    hot_cols = np.array([(f - 1 - yy) // c + 1 for yy in range(c)])     # columns k < f with k % c == y
    n_hot = rng.binomial(hot_cols[y], p_hi)
    n_cold = rng.binomial(f, p_lo, size=n)
    rows_h = np.repeat(np.arange(n, dtype=np.int64), n_hot)
    cols_h = y[rows_h].astype(np.int64) + c * (rng.random(rows_h.size) * hot_cols[y[rows_h]]).astype(np.int64)
    rows_c = np.repeat(np.arange(n, dtype=np.int64), n_cold)
    cols_c = rng.integers(0, f, size=rows_c.size, dtype=np.int64)
    keys = _sorted_unique(np.concatenate([rows_h * f + cols_h, rows_c * f + cols_c]))
    rows = keys // f
    ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=ptr[1:])
    return ptr, (keys % f).astype(np.int32), np.ones(keys.size, dtype=np.float32)


# NELL (the paper's headline sparse-feature dataset, Table: 65,755 nodes,
# 251,550 edges, 61,278 features, 186 classes, feature sparsity 99.21 %) with the paper's model
# (3 layers, hidden 32).  SURVEY §8(f) NEXT-2.  Features are produced as CSR.
CONFIGS["nell"] = WorkloadConfig("nell", 65755, 251550, (61278, 32, 32, 186), "binary_csr", 0.0079, 2.5, 0.2, 6)


def make_workload(name: str, feature_dtype=np.float32):
    """Return dict(src, dst, X, y, cfg) for one of CONFIGS (X_csr instead of X for CSR kinds)."""
    cfg = CONFIGS[name]
    y = make_labels(cfg.num_nodes, cfg.num_classes)
    src, dst = make_graph(cfg.num_nodes, cfg.nnz_a, cfg.num_classes, cfg.alpha, cfg.mu, cfg.seed)
    if cfg.feature_kind == "binary_csr":
        csr = make_features_csr(cfg.num_nodes, cfg.num_features, y, cfg.num_classes, cfg.density, cfg.seed)
        return {"src": src, "dst": dst, "X": None, "X_csr": csr, "y": y, "cfg": cfg}
    x = make_features(cfg.num_nodes, cfg.num_features, y, cfg.num_classes, cfg.feature_kind, cfg.density, cfg.seed)
    return {"src": src, "dst": dst, "X": x.astype(feature_dtype, copy=False), "y": y, "cfg": cfg}


def make_small(n: int, nnz_a: int, f: int, c: int, kind: str = "dense", density: float = 1.0,
               alpha: float = 2.5, mu: float = 0.2, seed: int = 0):
    """A small custom workload (tests): same recipe at arbitrary sizes."""
    y = make_labels(n, c)
    src, dst = make_graph(n, nnz_a, c, alpha, mu, seed)
    x = make_features(n, f, y, c, kind, density, seed)
    return {"src": src, "dst": dst, "X": x, "y": y}


def make_sbm_toy(n: int = 60, p_in: float = 0.3, p_out: float = 0.02, noise: float = 0.1, seed: int = 0):
    """2-block SBM of SURVEY c.4 'Epoch loop' pin: one-hot block + noise features."""
    rng = np.random.Generator(np.random.PCG64(seed))
    y = np.zeros(n, np.int32)
    y[n // 2:] = 1
    iu, ju = np.triu_indices(n, 1)
    same = y[iu] == y[ju]
    keep = rng.random(iu.size) < np.where(same, p_in, p_out)
    src = iu[keep].astype(np.int32)
    dst = ju[keep].astype(np.int32)
    x = np.zeros((n, 2), np.float32)
    x[np.arange(n), y] = 1.0
    x += (rng.integers(-(1 << 10), 1 << 10, size=(n, 2)).astype(np.float32) * np.float32(noise / 1024.0))
    return {"src": src, "dst": dst, "X": x, "y": y}
