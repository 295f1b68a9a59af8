"""Plain FP64 definition of one GCN training epoch (Morphling hot path).

TEST INFRASTRUCTURE ONLY — see oracle/__init__.py.  Nothing here is blocked,
fused or reordered beyond what the cited definition states; numpy / scipy
primitives (matmul, sort, sparse matmul) serve as single steps.

Notation: A symmetric 0/1 adjacency without self loops,
Ã = A + I, d̃ = Ã·1, Â = D̃^{-1/2} Ã D̃^{-1/2}; layer ℓ maps F_{ℓ-1} -> F_ℓ.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np
import scipy.sparse as sp

__all__ = [
    "OracleError", "Graph", "graph_build", "a_hat_values", "a_hat_dense_from_csr",
    "aggregate", "aggregate_rows", "analyze_features", "FeatureAnalysis",
    "splitmix64_stream", "xavier_init", "philox4x32_10", "dropout_keep",
    "dropout_threshold", "tf32_rna", "bf16_rne", "forward", "softmax_ce", "backward", "adam_step", "train",
    "AGGREGATORS", "aggregate_scheme", "aggregate_max", "aggregate_max_backward",
    "connected_components", "partition_components", "partition_greedy", "partition_hierarchical", "relabel",
    "partition_stats",
    "OPTIMIZERS", "sgd_step", "adamw_step",
    "partition_1d", "localize", "LocalPlan", "GOLDEN", "prepare", "threads_used", "csr_matmul",
]

GOLDEN = 0x9E3779B97F4A7C15
_M64 = (1 << 64) - 1


class OracleError(ValueError):
    """Error with the C-ABI class name (SURVEY §8(b) error table)."""

    def __init__(self, code: str, msg: str):
        super().__init__(f"{code}: {msg}")
        self.code = code


# ---------------------------------------------------------------------------
# a0 — graph build.  SURVEY c.2 G1-G6; PAPER P:222 ("CSR ... once during
# initialization").  Readings Q2-Q4 (symmetrise, dedup, drop
# input self loops, add I).
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class Graph:
    num_nodes: int
    row_ptr: np.ndarray   # int64[N+1]
    col_idx: np.ndarray   # int32[nnz], ascending per row, diagonal included
    deg: np.ndarray       # int32[N] = d̃
    dinv: np.ndarray      # float32[N] = (float)(1/sqrt((double)d̃))  (G6 bit recipe)

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    @property
    def rows(self) -> np.ndarray:
        return np.repeat(np.arange(self.num_nodes, dtype=np.int64), np.diff(self.row_ptr))


def graph_build(src, dst, num_nodes: int) -> Graph:
    n = int(num_nodes)
    if n <= 0:
        raise OracleError("EDEGENERATE", "N = 0")                        # G1
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    if src.shape != dst.shape:
        raise OracleError("EINVAL", "src/dst length mismatch")
    if src.size and (src.min() < 0 or dst.min() < 0 or src.max() >= n or dst.max() >= n):
        raise OracleError("ERANGE", "node id outside [0, N)")            # G1
    off = src != dst                                                     # G2: drop self loops
    u = np.concatenate([src[off], dst[off]])                             # G2: symmetrise
    v = np.concatenate([dst[off], src[off]])
    diag = np.arange(n, dtype=np.int64)
    keys = np.concatenate([u * n + v, diag * n + diag])                  # G3: S ∪ I
    keys = np.sort(keys)                                                 # G4 (u,v) order
    if keys.size:                                                        # G2 dedup
        keep = np.empty(keys.size, dtype=bool)
        keep[0] = True
        np.not_equal(keys[1:], keys[:-1], out=keep[1:])
        keys = keys[keep]
    rows = keys // n
    cols = keys % n
    counts = np.bincount(rows, minlength=n).astype(np.int64)
    row_ptr = np.zeros(n + 1, dtype=np.int64)                            # G4
    np.cumsum(counts, out=row_ptr[1:])
    deg = counts.astype(np.int32)                                        # G5
    dinv = (1.0 / np.sqrt(deg.astype(np.float64))).astype(np.float32)   # G6
    return Graph(n, row_ptr, cols.astype(np.int32), deg, dinv)


def a_hat_values(g: Graph) -> np.ndarray:
    """â_e = 1/sqrt(d̃_u d̃_v) in FP64 for every CSR entry (G6; Q1)."""
    d = g.deg.astype(np.float64)
    return 1.0 / np.sqrt(d[g.rows] * d[g.col_idx.astype(np.int64)])


def _a_hat_csr(g: Graph) -> sp.csr_matrix:
    # built once per graph (a pure function of the graph; the graph is never mutated)
    A = getattr(g, "_a_hat", None)
    if A is None:
        A = sp.csr_matrix((a_hat_values(g), g.col_idx.astype(np.int64), g.row_ptr),
                          shape=(g.num_nodes, g.num_nodes))
        object.__setattr__(g, "_a_hat", A)
    return A


def prepare(g: Graph) -> None:
    """Build the graph's cached Â / Ã operators now (setup, the analogue of the CSR build)."""
    _a_hat_csr(g)


def threads_used() -> int:
    """Host threads the sparse products use (ORACLE_THREADS, default: all cores)."""
    return _threads()


def _threads() -> int:
    import os
    return max(1, int(os.environ.get("ORACLE_THREADS", os.cpu_count() or 1)))


def csr_matmul(A: sp.csr_matrix, P: np.ndarray) -> np.ndarray:
    """A·P for a CSR A, the output rows cut into contiguous chunks computed on host threads
    (scipy's CSR product releases the GIL).  Each output row is the same sum, in the same CSR
    order, as the single-threaded product: the result is bit-identical to `A @ P` (SURVEY
    §8(c) c.1 allows parallelism over output rows; no blocking or reordering of any sum)."""
    P = np.asarray(P)
    n = A.shape[0]
    t = min(_threads(), max(1, n // 4096))
    if t <= 1 or P.ndim != 2:
        return np.asarray(A @ P)
    from concurrent.futures import ThreadPoolExecutor
    cuts = [n * i // t for i in range(t + 1)]
    out = np.empty((n, P.shape[1]), dtype=np.result_type(A.dtype, P.dtype))

    def run(i):
        out[cuts[i]:cuts[i + 1]] = A[cuts[i]:cuts[i + 1]] @ P

    with ThreadPoolExecutor(t) as ex:
        list(ex.map(run, range(t)))
    return out


def a_hat_dense_from_csr(g: Graph) -> np.ndarray:
    return _a_hat_csr(g).toarray()


def aggregate(g: Graph, P: np.ndarray) -> np.ndarray:
    """Y = Â·P in FP64 (F2 / B2).  Alg. 3 P:373-384 computes the same sum
    Y[u,f] = Σ_{ei∈row u} val[ei]·X[col[ei], f]; here val = â (Q1)."""
    P = np.asarray(P, dtype=np.float64)
    return csr_matmul(_a_hat_csr(g), P)


def aggregate_rows(g: Graph, P: np.ndarray, rows) -> np.ndarray:
    """Â·P for a subset of output rows, one row at a time (full-size sampling)."""
    d = g.deg.astype(np.float64)
    out = np.zeros((len(rows), P.shape[1]), dtype=np.float64)
    for i, u in enumerate(rows):
        s, e = int(g.row_ptr[u]), int(g.row_ptr[u + 1])
        cols = g.col_idx[s:e].astype(np.int64)
        w = 1.0 / np.sqrt(d[u] * d[cols])
        out[i] = w @ np.asarray(P[cols], dtype=np.float64)
    return out


# ---------------------------------------------------------------------------
# Other aggregation schemes: "GCN uses normalized mean aggregation ...
# GIN employs sum aggregation"; "multiple aggregation schemes (mean, max, sum)";
# Listing 1's SAGE "Max".  Readings R6-R8: every scheme aggregates over
# Ñ(u) = N(u) ∪ {u}, the same Ã = A + I the GCN uses (Q2); max is taken before the transform
# (P:92 applies W to AGGREGATE(h)); ties go to the smallest node id.
# ---------------------------------------------------------------------------
AGGREGATORS = ("gcn", "sum", "mean", "max")


def _a_tilde_csr(g: Graph) -> sp.csr_matrix:
    """Ã = A + I as a 0/1 CSR (the graph's pattern, diagonal included)."""
    A = getattr(g, "_a_tilde", None)
    if A is None:
        A = sp.csr_matrix((np.ones(g.nnz), g.col_idx.astype(np.int64), g.row_ptr),
                          shape=(g.num_nodes, g.num_nodes))
        object.__setattr__(g, "_a_tilde", A)
    return A


def aggregate_scheme(g: Graph, P: np.ndarray, scheme: str, transpose: bool = False) -> np.ndarray:
    """Linear aggregations in FP64: gcn Â·P; sum Ã·P; mean D̃^{-1}Ã·P.  transpose=True applies
    the adjoint used by the backward pass (Âᵀ = Â, Ãᵀ = Ã, (D̃^{-1}Ã)ᵀ = Ã·D̃^{-1})."""
    P = np.asarray(P, dtype=np.float64)
    if scheme == "gcn":
        return aggregate(g, P)
    At = _a_tilde_csr(g)
    if scheme == "sum":
        return csr_matmul(At, P)
    if scheme == "mean":
        d = g.deg.astype(np.float64)[:, None]
        return csr_matmul(At, P / d) if transpose else csr_matmul(At, P) / d
    raise ValueError(f"not a linear aggregation scheme: {scheme}")


def aggregate_max(g: Graph, P: np.ndarray):
    """Y[u,c] = max over v in Ñ(u) of P[v,c]; arg[u,c] = the smallest such v (ties, R7).
    Plain per-row loop: the row's neighbour ids are ascending, so np.argmax's first maximum is
    the smallest id."""
    P = np.asarray(P, dtype=np.float64)
    n, f = P.shape
    Y = np.empty((n, f), dtype=np.float64)
    arg = np.empty((n, f), dtype=np.int64)
    cols_f = np.arange(f)
    for u in range(n):
        nb = g.col_idx[g.row_ptr[u]:g.row_ptr[u + 1]].astype(np.int64)
        block = P[nb]
        k = np.argmax(block, axis=0)
        Y[u] = block[k, cols_f]
        arg[u] = nb[k]
    return Y, arg


def aggregate_max_backward(dY: np.ndarray, arg: np.ndarray, num_nodes: int) -> np.ndarray:
    """Adjoint of aggregate_max: every dY[u,c] is routed to its argmax node arg[u,c]."""
    dY = np.asarray(dY, dtype=np.float64)
    dH = np.zeros((num_nodes, dY.shape[1]), dtype=np.float64)
    np.add.at(dH, (arg, np.broadcast_to(np.arange(dY.shape[1]), arg.shape)), dY)
    return dH


# ---------------------------------------------------------------------------
# a1 — feature analysis and the dense/sparse switch.  Alg. 1 Initialize
# P:256-266; Eq. 1; τ≈0.80 P:216; readings Q11, Q12, Q28.
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class FeatureAnalysis:
    nnz: int
    mode: int              # 0 Dense, 1 Sparse
    is_binary: bool
    sparsity: float        # s = 1 - nnz/(N*F)
    csr: tuple | None      # (ptr int64[N+1], idx int32[nnz], val f32[nnz])
    csc: tuple | None      # (ptr int64[F+1], idx int32[nnz] rows ascending, val f32[nnz])


def analyze_features(X, tau_bp: int = 8000, force_mode: int = -1) -> FeatureAnalysis:
    if sp.issparse(X):  # CSR input (NELL-scale features): the same S1-S3 on the stored entries
        X = sp.csr_matrix(X, dtype=np.float32)
        n, f = X.shape
        if n * f == 0:
            raise OracleError("EDEGENERATE", "N*F = 0")
        keep = X.data != np.float32(0.0)                                        # S1
        rows = np.repeat(np.arange(n), np.diff(X.indptr))[keep]
        cols = X.indices[keep].astype(np.int64)
        vals = X.data[keep]
        order = np.lexsort((cols, rows))
        rows, cols, vals = rows[order], cols[order], vals[order]
        nnz = int(vals.size)
        sparse = 10000 * nnz <= (10000 - int(tau_bp)) * n * f                  # S2
        mode = int(sparse) if force_mode < 0 else int(force_mode)
        csr = csc = None
        if mode == 1:                                                          # S3
            ptr = np.zeros(n + 1, np.int64)
            np.cumsum(np.bincount(rows, minlength=n), out=ptr[1:])
            csr = (ptr, cols.astype(np.int32), vals.astype(np.float32))
            o2 = np.lexsort((rows, cols))
            cptr = np.zeros(f + 1, np.int64)
            np.cumsum(np.bincount(cols, minlength=f), out=cptr[1:])
            csc = (cptr, rows[o2].astype(np.int32), vals[o2].astype(np.float32))
        return FeatureAnalysis(nnz, mode, bool(np.all(vals == np.float32(1.0))), 1.0 - nnz / (n * f), csr, csc)
    X = np.asarray(X, dtype=np.float32)
    n, f = X.shape
    if n * f == 0:
        raise OracleError("EDEGENERATE", "N*F = 0")
    nz = X != np.float32(0.0)                                   # S1 (IEEE compare, Q12)
    nnz = int(nz.sum())
    sparse = 10000 * nnz <= (10000 - int(tau_bp)) * n * f       # S2: s >= τ, integer-decided
    mode = int(sparse) if force_mode < 0 else int(force_mode)
    s = 1.0 - nnz / (n * f)
    is_binary = bool(np.all(X[nz] == np.float32(1.0)))
    csr = csc = None
    if mode == 1:                                               # S3
        r, c = np.nonzero(nz)                                   # row-major order
        ptr = np.zeros(n + 1, np.int64)
        np.cumsum(np.bincount(r, minlength=n), out=ptr[1:])
        csr = (ptr, c.astype(np.int32), X[r, c].astype(np.float32))
        ct, rt = np.nonzero(nz.T)                               # column-major, rows ascending
        cptr = np.zeros(f + 1, np.int64)
        np.cumsum(np.bincount(ct, minlength=f), out=cptr[1:])
        csc = (cptr, rt.astype(np.int32), X[rt, ct].astype(np.float32))
    return FeatureAnalysis(nnz, mode, is_binary, s, csr, csc)


# ---------------------------------------------------------------------------
# Xavier initialisation ("xaviers", Listing 1; bound S:322; stream Q16)
# ---------------------------------------------------------------------------
def splitmix64_stream(seed: int, count: int) -> np.ndarray:
    """The splitmix64 sequence, written out sequentially (Q16)."""
    out = np.empty(count, dtype=np.uint64)
    state = seed & _M64
    for i in range(count):
        state = (state + GOLDEN) & _M64
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        out[i] = z ^ (z >> 31)
    return out


def xavier_init(dims, seed: int):
    """W_ℓ ~ U(-a, a), a = sqrt(6/(f_in+f_out)) on unpadded fans; b_ℓ = 0 (Q6, Q16).

    Stream for layer ℓ (1-based): splitmix64 seeded seed ^ (ℓ·GOLDEN mod 2^64),
    row-major fill of [f_in, f_out]; value a·(2·(x>>40)/2^24 − 1) in double,
    rounded once to f32.
    """
    Ws, bs = [], []
    for l in range(1, len(dims)):
        fi, fo = int(dims[l - 1]), int(dims[l])
        a = math.sqrt(6.0 / (fi + fo))
        x = splitmix64_stream(seed ^ ((l * GOLDEN) & _M64), fi * fo)
        u24 = (x >> np.uint64(40)).astype(np.float64)
        w = a * (2.0 * u24 / float(1 << 24) - 1.0)
        Ws.append(w.astype(np.float32).reshape(fi, fo))
        bs.append(np.zeros(fo, dtype=np.float32))
    return Ws, bs


# ---------------------------------------------------------------------------
# Dropout mask (Q10): Philox4x32-10, key=(seed lo, seed hi),
# counter=(row, col/4, layer, epoch), lane col%4; keep iff u32 >= floor(p·2^32).
# ---------------------------------------------------------------------------
_PM0, _PM1 = 0xD2511F53, 0xCD9E8D57
_PW0, _PW1 = 0x9E3779B9, 0xBB67AE85


def philox4x32_10(ctr, key):
    """Philox4x32 with 10 rounds (Salmon et al. 2011, Random123); vectorised over
    leading axes: ctr uint64-able [...,4], key [...,2]; returns uint32 [...,4]."""
    c = [np.asarray(ctr[..., i], dtype=np.uint64) & np.uint64(0xFFFFFFFF) for i in range(4)]
    k0 = np.asarray(key[..., 0], dtype=np.uint64) & np.uint64(0xFFFFFFFF)
    k1 = np.asarray(key[..., 1], dtype=np.uint64) & np.uint64(0xFFFFFFFF)
    mask = np.uint64(0xFFFFFFFF)
    for r in range(10):
        if r > 0:
            k0 = (k0 + np.uint64(_PW0)) & mask
            k1 = (k1 + np.uint64(_PW1)) & mask
        p0 = np.uint64(_PM0) * c[0]
        p1 = np.uint64(_PM1) * c[2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & mask
        hi1, lo1 = p1 >> np.uint64(32), p1 & mask
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
    return np.stack([x.astype(np.uint32) for x in c], axis=-1)


def dropout_threshold(p: float) -> int:
    return int(math.floor(float(np.float32(p)) * 4294967296.0))


def dropout_keep(n_rows: int, n_cols: int, p: float, seed: int, layer: int, epoch: int,
                 row0: int = 0) -> np.ndarray:
    """Boolean keep mask [n_rows, n_cols] for hidden layer `layer` at `epoch` (Q10)."""
    rows = np.arange(row0, row0 + n_rows, dtype=np.uint64)
    cols = np.arange(n_cols, dtype=np.uint64)
    ctr = np.zeros((n_rows, n_cols, 4), dtype=np.uint64)
    ctr[..., 0] = rows[:, None]
    ctr[..., 1] = (cols // np.uint64(4))[None, :]
    ctr[..., 2] = np.uint64(layer)
    ctr[..., 3] = np.uint64(epoch)
    key = np.zeros((n_rows, n_cols, 2), dtype=np.uint64)
    key[..., 0] = np.uint64(seed & 0xFFFFFFFF)
    key[..., 1] = np.uint64((seed >> 32) & 0xFFFFFFFF)
    out = philox4x32_10(ctr, key)
    lane = (cols % np.uint64(4)).astype(np.int64)
    u32 = np.take_along_axis(out, np.broadcast_to(lane[None, :, None], (n_rows, n_cols, 1)), axis=2)[..., 0]
    return u32.astype(np.uint64) >= np.uint64(dropout_threshold(p))


# ---------------------------------------------------------------------------
# Forward (c.2 F1-F4): layer update of P:92 with Q1 (Â), Q6 (bias),
# Q8 (ReLU hidden, identity output), Q10 (dropout after ReLU).
# ---------------------------------------------------------------------------
def tf32_rna(x) -> np.ndarray:
    """TF32 operand rounding (reading R2; north_star "TF32 in, FP32 accumulate"): the value as an
    fp32 number with its 23-bit mantissa rounded to TF32's 10 bits, to nearest, ties away from
    zero (PTX cvt.rna.tf32.f32).  Sign-magnitude layout: adding half an ulp (bit 12) to the
    magnitude bits and clearing the low 13 bits rounds |x| half-up.  Finite inputs only."""
    a = np.array(x, dtype=np.float32, copy=True)
    u = a.view(np.uint32)
    u += np.uint32(0x1000)
    u &= np.uint32(0xFFFFE000)
    return a.astype(np.float64)


def bf16_rne(x) -> np.ndarray:
    """BF16 operand rounding (north_star "TF32 or BF16 inputs, FP32 accumulate"): the value as an
    fp32 number with its mantissa rounded to BF16's 7 bits, to nearest, ties to even (the
    cvt.rn.bf16.f32 rule): add 0x7FFF plus the lowest kept bit, clear the low 16 bits.  Finite
    inputs only."""
    a = np.array(x, dtype=np.float32, copy=True)
    u = a.view(np.uint32)
    u += np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))
    u &= np.uint32(0xFFFF0000)
    return a.astype(np.float64)


def _operand(M, rounding):
    """A dense GEMM operand as the tensor core sees it (identity unless rounding is "tf32" or
    "bf16")."""
    if rounding is None or sp.issparse(M):
        return M
    if rounding == "tf32":
        return tf32_rna(M)
    if rounding == "bf16":
        return bf16_rne(M)
    raise ValueError(rounding)


def forward(g: Graph, X, Ws, bs, dropout_p: float = 0.0, seed: int = 0, epoch: int = 1, operand_rounding=None,
            aggregator: str = "gcn", orders=None):
    # X may be a scipy CSR matrix (sparse features): X·W_1 and X^T·G are then sparse products.
    # operand_rounding="tf32" rounds both operands of every dense product H·W (R2); sparse products
    # (X_csr·W_1) and the aggregation stay exact.  It models transform-first layers.
    # aggregator: "gcn" (Â, the north star), "sum", "mean" (linear: Z = AGG(H·W) + b) or "max"
    # (Z = MAX(H)·W + b, R7); see aggregate_scheme / aggregate_max.
    # orders: per layer "TF" (transform first, Z = AGG(H·W) + b, the default) or "AF" (aggregate
    # first, Z = AGG(H)·W + b) — the same Z in exact arithmetic (AGG is linear, P:88 / reading Q7);
    # the order only decides which operand a rounded product sees (operand_rounding: AF rounds
    # Y = AGG(H), TF rounds H).
    if aggregator not in AGGREGATORS:
        raise ValueError(aggregator)
    orders = tuple(orders) if orders is not None else ("TF",) * len(Ws)
    if len(orders) != len(Ws) or any(o not in ("TF", "AF") for o in orders):
        raise ValueError(orders)
    H = X.astype(np.float64).tocsr() if sp.issparse(X) else np.asarray(X, dtype=np.float64)
    hs, zs, ys, args = [H], [], [], []
    L = len(Ws)
    r = operand_rounding
    for l in range(1, L + 1):
        W = np.asarray(Ws[l - 1], dtype=np.float64)
        if aggregator == "max":
            # F2 before F1 (R7).  With operand_rounding the max is taken on the operand as the
            # kernel stores it (TF32): an argmax is decided in the kernel's precision
            Y, arg = aggregate_max(g, _operand(H.toarray() if sp.issparse(H) else H, r))
            ys.append(Y)
            args.append(arg)
            Z = _operand(Y, r) @ _operand(W, r) + np.asarray(bs[l - 1], dtype=np.float64)
        elif orders[l - 1] == "AF":
            if sp.issparse(H):
                raise ValueError("aggregate-first needs dense features")
            Y = aggregate_scheme(g, H, aggregator)                       # F2 before F1 (Q7)
            ys.append(Y)
            Z = _operand(Y, r) @ _operand(W, r) + np.asarray(bs[l - 1], dtype=np.float64)
        else:
            ys.append(None)
            P = _operand(H, r) @ (W if sp.issparse(H) else _operand(W, r))   # F1
            Z = aggregate_scheme(g, P, aggregator) + np.asarray(bs[l - 1], dtype=np.float64)   # F2
        zs.append(Z)
        if l < L:
            H = np.maximum(Z, 0.0)                                       # F3
            if dropout_p > 0.0:
                keep = dropout_keep(Z.shape[0], Z.shape[1], dropout_p, seed, l, epoch)
                H = H * keep / (1.0 - float(np.float32(dropout_p)))
            hs.append(H)
    return zs[-1], {"H": hs, "Z": zs, "dropout_p": dropout_p, "seed": seed, "epoch": epoch, "rounding": r,
                    "aggregator": aggregator, "Y": ys, "arg": args, "orders": orders}


def softmax_ce(Z, labels, mask=None, n_lab: int | None = None):
    """L1-L3 (Q9, Q17, Q25): mean softmax cross-entropy over labelled rows."""
    Z = np.asarray(Z, dtype=np.float64)
    labels = np.asarray(labels, dtype=np.int64)
    lab = np.ones(Z.shape[0], bool) if mask is None else np.asarray(mask, bool)
    nl = int(lab.sum()) if n_lab is None else int(n_lab)
    m = Z.max(axis=1)
    lse = m + np.log(np.exp(Z - m[:, None]).sum(axis=1))               # L1
    rows = np.nonzero(lab)[0]
    loss = float((lse[rows] - Z[rows, labels[rows]]).sum() / nl)        # L2
    dZ = np.exp(Z - lse[:, None])
    dZ[np.arange(Z.shape[0]), labels] -= 1.0
    dZ /= nl                                                             # L3
    dZ[~lab] = 0.0
    return loss, dZ


def backward(g: Graph, cache, Ws, dZ):
    """B1-B4: returns (dWs, dbs).  The upstream gradient of every layer, dZ_l = ∂loss/∂Z_l, is
    recorded in cache["dZ"][l-1], and the gradient w.r.t. the hidden activation before the ReLU
    mask, dH_l = ∂loss/∂H_l, in cache["dH"][l-1] for l < L (outputs for bounds in tests; no extra
    arithmetic)."""
    L = len(Ws)
    dWs, dbs = [None] * L, [None] * L
    agg = cache.get("aggregator", "gcn")
    cache["dZ"] = [None] * L
    cache["dH"] = [None] * L
    for l in range(L, 0, -1):
        cache["dZ"][l - 1] = dZ
        dbs[l - 1] = dZ.sum(axis=0)                                     # B1
        r = cache.get("rounding")
        W = np.asarray(Ws[l - 1], dtype=np.float64)
        if agg == "max":                                                 # Z = Y·W + b, Y = MAX(H)
            dWs[l - 1] = _operand(cache["Y"][l - 1], r).T @ _operand(dZ, r)
            if l > 1:
                dY = _operand(dZ, r) @ _operand(W, r).T
                dH = aggregate_max_backward(dY, cache["arg"][l - 1], g.num_nodes)
        elif cache.get("orders", ("TF",) * L)[l - 1] == "AF":           # Z = Y·W + b, Y = AGG(H)
            dWs[l - 1] = _operand(cache["Y"][l - 1], r).T @ _operand(dZ, r)
            if l > 1:
                dH = aggregate_scheme(g, _operand(dZ, r) @ _operand(W, r).T, agg, transpose=True)
        else:
            G = aggregate_scheme(g, dZ, agg, transpose=True)             # B2 (Âᵀ = Â)
            Hp = cache["H"][l - 1]
            dWs[l - 1] = _operand(Hp, r).T @ (G if sp.issparse(Hp) else _operand(G, r))   # B3
            if l > 1:
                dH = _operand(G, r) @ _operand(W, r).T                   # B4
        if l > 1:
            cache["dH"][l - 2] = dH
            dZ = dH * (cache["Z"][l - 2] > 0.0)                          # ReLU'(0) := 0 (Q8)
            if cache["dropout_p"] > 0.0:
                keep = dropout_keep(dZ.shape[0], dZ.shape[1], cache["dropout_p"], cache["seed"],
                                    l - 1, cache["epoch"])
                dZ = dZ * keep / (1.0 - float(np.float32(cache["dropout_p"])))
    return dWs, dbs


def adam_step(params, grads, m, v, t: int, lr=0.01, beta1=0.9, beta2=0.999, eps=1e-8):
    """A1 (P:170 lr/β1/β2, Q15 ε outside sqrt, bias-corrected, t from 1). In place."""
    for p, gr, mm, vv in zip(params, grads, m, v):
        mm *= beta1
        mm += (1.0 - beta1) * gr
        vv *= beta2
        vv += (1.0 - beta2) * gr * gr
        mhat = mm / (1.0 - beta1 ** t)
        vhat = vv / (1.0 - beta2 ** t)
        p -= lr * mhat / (np.sqrt(vhat) + eps)


def sgd_step(params, grads, vel, lr=0.01, momentum=0.0, weight_decay=0.0):
    """SGD (reading R8, the common definition): g' = g + wd·p; with momentum μ > 0 the
    velocity is v = μ·v + g' (v = g' at the first step, i.e. v starts at zero); p -= lr·v
    (p -= lr·g' when μ = 0).  In place."""
    for p, gr, vv in zip(params, grads, vel):
        d = gr + weight_decay * p if weight_decay != 0.0 else gr
        if momentum != 0.0:
            vv *= momentum
            vv += d
            d = vv
        p -= lr * d


def adamw_step(params, grads, m, v, t: int, lr=0.01, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01):
    """AdamW ("applies decoupled weight decay before the Adam update"):
    p ← p − lr·wd·p, then adam_step.  In place."""
    for p in params:
        p -= lr * weight_decay * p
    adam_step(params, grads, m, v, t, lr, beta1, beta2, eps)


OPTIMIZERS = ("adam", "sgd", "adamw")


def train(g: Graph, X, labels, dims, epochs: int, seed: int = 42, lr=0.01, beta1=0.9,
          beta2=0.999, eps=1e-8, mask=None, dropout_p: float = 0.0, dropout_seed: int = 0,
          init=None, operand_rounding=None, aggregator: str = "gcn", optimizer: str = "adam",
          weight_decay: float = 0.0, momentum: float = 0.0, orders=None):
    """Epoch loop (Listing 1): loss_t at θ_{t-1}, backward, optimizer -> θ_t
    (Adam by default; SGD / AdamW)."""
    if optimizer not in OPTIMIZERS:
        raise ValueError(optimizer)
    if init is None:
        Ws, bs = xavier_init(dims, seed)
    else:
        Ws, bs = init
    params = [np.asarray(w, np.float64).copy() for w in Ws] + [np.asarray(b, np.float64).copy() for b in bs]
    L = len(Ws)
    m = [np.zeros_like(p) for p in params]
    v = [np.zeros_like(p) for p in params]
    losses = []
    for t in range(1, epochs + 1):
        Z, cache = forward(g, X, params[:L], params[L:], dropout_p, dropout_seed, t, operand_rounding, aggregator,
                           orders)
        loss, dZ = softmax_ce(Z, labels, mask)
        losses.append(loss)
        dWs, dbs = backward(g, cache, params[:L], dZ)
        if optimizer == "adam":
            adam_step(params, dWs + dbs, m, v, t, lr, beta1, beta2, eps)
        elif optimizer == "adamw":
            adamw_step(params, dWs + dbs, m, v, t, lr, beta1, beta2, eps, weight_decay)
        else:
            sgd_step(params, dWs + dbs, m, lr, momentum, weight_decay)
    return losses, params


# ---------------------------------------------------------------------------
# Distributed plans (c.2 D1-D5): 1D contiguous partition balanced by Σ d̃
# (Phase III weight deg+1, Alg. 4; Q20), G2L local-then-ghost layout
# (P:514-515), halo lists (Q21).
# ---------------------------------------------------------------------------
def partition_1d(row_ptr, world: int) -> np.ndarray:
    """bounds[r] = min{u in [0,N] : world·row_ptr[u] >= r·nnz} (D1)."""
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    nnz = int(row_ptr[-1])
    bounds = np.empty(world + 1, dtype=np.int64)
    u = 0
    for r in range(world + 1):
        while world * int(row_ptr[u]) < r * nnz:
            u += 1
        bounds[r] = u
    return bounds


# ---------------------------------------------------------------------------
# Alg. 4: Phase II component bin packing and Phase III
# load-aware greedy, then a relabelling that makes every rank's nodes a contiguous id range
# so the 1D machinery above (bounds, G2L, halo lists) applies unchanged.  Phase I (METIS) is
# out of scope.  Reading R9: ties in every sort / argmin go to the smaller node id / lower rank.
# ---------------------------------------------------------------------------
def connected_components(g: Graph):
    """Component id per node by BFS over A ("detects ... connected components via BFS"),
    ids numbered in order of each component's smallest node."""
    n = g.num_nodes
    comp = np.full(n, -1, dtype=np.int64)
    c = 0
    for s in range(n):
        if comp[s] >= 0:
            continue
        comp[s] = c
        queue = [s]
        while queue:
            u = queue.pop()
            for v in g.col_idx[g.row_ptr[u]:g.row_ptr[u + 1]]:
                if comp[v] < 0:
                    comp[v] = c
                    queue.append(int(v))
        c += 1
    return comp, c


def partition_components(g: Graph, world: int):
    """Phase II (Alg. 4 lines "Sort Comps by size descending ... p = argmin(Weights) ...
    Weights[p] += |C|").  Returns (part, n_components); part is None for a connected graph (the
    algorithm falls through to Phase III)."""
    comp, nc = connected_components(g)
    if nc <= 1:
        return None, nc
    sizes = np.bincount(comp, minlength=nc)
    order = sorted(range(nc), key=lambda c: (-int(sizes[c]), c))     # size desc, then first node
    weights = [0] * world
    part = np.empty(g.num_nodes, dtype=np.int32)
    for c in order:
        p = min(range(world), key=lambda q: (weights[q], q))
        part[comp == c] = p
        weights[p] += int(sizes[c])
    return part, nc


def partition_greedy(g: Graph, world: int) -> np.ndarray:
    """Phase III (Alg. 4: "Sort V by Degree descending ... p = argmin(Weights); Weights[p] +=
    deg(v) + 1"); deg(v) = |N(v)| in A, so deg(v) + 1 = d̃_v."""
    d = g.deg.astype(np.int64) - 1
    order = sorted(range(g.num_nodes), key=lambda v: (-int(d[v]), v))
    weights = [0] * world
    part = np.empty(g.num_nodes, dtype=np.int32)
    for v in order:
        p = min(range(world), key=lambda q: (weights[q], q))
        part[v] = p
        weights[p] += int(d[v]) + 1
    return part


PHASE2_BALANCE_PCT = 105   # reading R10: Phase II is kept iff max bin ≤ 1.05 · mean and no bin is empty


def partition_hierarchical(g: Graph, world: int):
    """Alg. 4 without Phase I: Phase II when the graph is disconnected AND its bin packing is
    balanced (every bin non-empty, max load ≤ 1.05·mean in |C| units, decided in integers:
    100·world·max ≤ 105·N), else Phase III (a giant component or fewer components than ranks
    falls through, reading R10).  Returns (part, phase)."""
    part, nc = partition_components(g, world)
    if part is not None:
        loads = np.bincount(part, minlength=world)
        if loads.min() > 0 and 100 * world * int(loads.max()) <= PHASE2_BALANCE_PCT * g.num_nodes:
            return part, 2
    return partition_greedy(g, world), 3


def relabel(part, world: int):
    """New ids: rank 0's nodes first, then rank 1's, ..., each rank's in ascending old id.
    Returns (new_id[old], bounds[world+1]) so rank r owns new ids [bounds[r], bounds[r+1])."""
    part = np.asarray(part, dtype=np.int64)
    n = part.size
    order = np.lexsort((np.arange(n), part))
    new_id = np.empty(n, dtype=np.int64)
    new_id[order] = np.arange(n)
    bounds = np.zeros(world + 1, dtype=np.int64)
    np.cumsum(np.bincount(part, minlength=world), out=bounds[1:])
    return new_id, bounds


def partition_stats(g: Graph, part, world: int) -> np.ndarray:
    """Per rank [owned nodes, Σ d̃ (the SpMM work, T_comp ∝ Σ deg·F), distinct ghost
    nodes (halo rows received per exchange), cut entries (nonzeros of A whose column
    lives on another rank)]."""
    part = np.asarray(part, dtype=np.int64)
    rows = g.rows
    cols = g.col_idx.astype(np.int64)
    out = np.zeros((world, 4), dtype=np.int64)
    for r in range(world):
        mine = part == r
        out[r, 0] = int(mine.sum())
        out[r, 1] = int(g.deg[mine].astype(np.int64).sum())
        sel = mine[rows] & (part[cols] != r)
        out[r, 2] = int(np.unique(cols[sel]).size)
        out[r, 3] = int(sel.sum())
    return out


@dataclasses.dataclass
class LocalPlan:
    rank: int
    n_own: int
    row0: int
    ghosts: np.ndarray        # int64 global ids, ascending (D2)
    row_ptr: np.ndarray       # int64[n_own+1] local CSR
    col_idx: np.ndarray       # int32 local ids, [owned | ghosts] per row (D3)
    split: np.ndarray         # int64[n_own]: index in the row where ghost columns start
    recv_offset: np.ndarray   # int64[world]: offset of peer q's slice inside the ghost region
    n_recv: np.ndarray        # int64[world]
    send_ids: list            # per peer: ascending owned LOCAL ids to send (D4)


def localize(g: Graph, bounds, rank: int) -> LocalPlan:
    bounds = np.asarray(bounds, dtype=np.int64)
    world = len(bounds) - 1
    b0, b1 = int(bounds[rank]), int(bounds[rank + 1])
    n_own = b1 - b0
    s, e = int(g.row_ptr[b0]), int(g.row_ptr[b1])
    cols = g.col_idx[s:e].astype(np.int64)
    is_ghost = (cols < b0) | (cols >= b1)
    ghosts = np.unique(cols[is_ghost])                                   # D2
    lid = np.where(is_ghost, n_own + np.searchsorted(ghosts, cols), cols - b0)   # D3
    local_rp = g.row_ptr[b0:b1 + 1] - s
    new_cols = np.empty_like(lid)
    split = np.empty(n_own, dtype=np.int64)
    for i in range(n_own):
        a, b = int(local_rp[i]), int(local_rp[i + 1])
        row = np.sort(lid[a:b])
        new_cols[a:b] = row
        split[i] = int((row < n_own).sum())
    owner = np.searchsorted(bounds, ghosts, side="right") - 1
    n_recv = np.bincount(owner, minlength=world).astype(np.int64)
    recv_offset = np.zeros(world, dtype=np.int64)
    np.cumsum(n_recv[:-1], out=recv_offset[1:])
    send_ids = []
    for q in range(world):
        if q == rank:
            send_ids.append(np.zeros(0, dtype=np.int64))
            continue
        q0, q1 = int(bounds[q]), int(bounds[q + 1])
        qs, qe = int(g.row_ptr[q0]), int(g.row_ptr[q1])
        qc = g.col_idx[qs:qe].astype(np.int64)
        need = np.unique(qc[(qc >= b0) & (qc < b1)])                    # D4
        send_ids.append(need - b0)
    return LocalPlan(rank, n_own, b0, ghosts, local_rp.astype(np.int64), new_cols.astype(np.int32),
                     split, recv_offset, n_recv, send_ids)
