"""Python API over the C-ABI (marshalling only; every step runs in libmorphling.so kernels).

    g = Graph(src, dst, num_nodes)                         # a0, mph_graph_build
    f = Features(X_cuda)                                   # a1, mph_features_create (tau: B200 value)
    m = GCN(g, f, dims=(602, 128, 41))                     # mph_gcn_create
    m.init_xavier(42); m.set_labels(y_cuda)
    loss = m.train_epoch(t=1)                              # a2..a11 + Adam, loss in a device double

torch is used for device memory and streams only.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib as L
from ._lib import AdamCfg, Epilogue, GcnDesc, MorphlingError, OptimCfg  # noqa: F401

DEFAULT_ADAM = (0.01, 0.9, 0.999, 1e-8)  # Listing 1; eps reading Q15


def optimizer(kind: str = "adam", lr: float = 0.01, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
              weight_decay: float = 0.0, momentum: float = 0.0) -> OptimCfg:
    """mph_optim_cfg for "adam" | "sgd" | "adamw" (reading R8)."""
    return OptimCfg(L.OPT[kind], lr, beta1, beta2, eps, weight_decay, momentum)


def pad_width(w: int) -> int:
    return 4 if w <= 4 else (w + 7) // 8 * 8


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


class _CAI:
    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


_TYPESTR = {torch.float32: "<f4", torch.float64: "<f8", torch.int32: "<i4", torch.int64: "<i8", torch.uint8: "|u1",
            torch.int16: "<i2"}


def device_view(ptr: int, shape, dtype) -> torch.Tensor:
    """Zero-copy torch view of library-owned device memory (borrowed: valid until the handle dies)."""
    if int(np.prod(shape)) == 0 or not ptr:
        return torch.empty(shape, dtype=dtype, device="cuda")
    return torch.as_tensor(_CAI(ptr, shape, _TYPESTR[dtype]), device="cuda")


def _destroy(fn_name: str, h):
    """Release a handle; a no-op during interpreter teardown (module globals already cleared)."""
    fn = getattr(L, fn_name, None)
    if callable(fn):
        fn(h)


def _out_ptr():
    return C.c_void_p()


class Graph:
    """a0 — CSR of Â's pattern (symmetrised, deduplicated, self loops added) + deg + dinv."""

    def __init__(self, src=None, dst=None, num_nodes: int = 0, stream=None, _handle=None):
        if _handle is not None:
            self.h = _handle
        else:
            src = np.ascontiguousarray(np.asarray(src, dtype=np.int32))
            dst = np.ascontiguousarray(np.asarray(dst, dtype=np.int32))
            h = _out_ptr()
            L.mph_graph_build(src.ctypes.data, dst.ctypes.data, int(src.size), int(num_nodes), stream_ptr(stream),
                              C.byref(h))
            self.h = h
        nr, nc, nnz, md = C.c_int32(), C.c_int32(), C.c_int64(), C.c_int32()
        L.mph_graph_info(self.h, C.byref(nr), C.byref(nc), C.byref(nnz), C.byref(md))
        self.n_rows, self.n_cols, self.nnz, self.max_deg = nr.value, nc.value, nnz.value, md.value

    @classmethod
    def from_plan(cls, plan: "Plan", stream=None) -> "Graph":
        h = _out_ptr()
        L.mph_graph_from_plan(plan.h, stream_ptr(stream), C.byref(h))
        g = cls(_handle=h)
        g.world, g.rank = plan.world, plan.rank
        return g

    def localize(self, bounds: np.ndarray, rank: int, stream=None) -> "Graph":
        """mph_graph_localize: rank's owned+ghost view of this global graph (D1-D4)."""
        b = np.ascontiguousarray(bounds, dtype=np.int64)
        h = _out_ptr()
        L.mph_graph_localize(self.h, b.ctypes.data, int(b.size - 1), int(rank), stream_ptr(stream), C.byref(h))
        g = Graph(_handle=h)
        g.world, g.rank = int(b.size - 1), int(rank)
        return g

    def halo_plan(self, peer: int) -> dict:
        """mph_halo_plan of a localized graph: send ids (device view), recv offset and count."""
        ids, ns, ro, nr = C.c_void_p(), C.c_int64(), C.c_int64(), C.c_int64()
        L.mph_halo_plan(self.h, int(peer), C.byref(ids), C.byref(ns), C.byref(ro), C.byref(nr))
        return {"send_ids": device_view(ids.value, (ns.value,), torch.int32), "recv_offset": ro.value,
                "n_recv": nr.value}

    def csr(self):
        rp, ci, dg, di = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
        L.mph_graph_csr(self.h, C.byref(rp), C.byref(ci), C.byref(dg), C.byref(di))
        return (device_view(rp.value, (self.n_rows + 1,), torch.int64),
                device_view(ci.value, (self.nnz,), torch.int32),
                device_view(dg.value, (self.n_cols,), torch.int32),
                device_view(di.value, (self.n_cols,), torch.float32))

    @property
    def dinv(self) -> torch.Tensor:
        return self.csr()[3]

    def spmm(self, inp: torch.Tensor, out: torch.Tensor, w: int | None = None, epi: Epilogue | None = None,
             part: int = -1, stream=None):
        w = inp.shape[1] if w is None else w
        e = C.byref(epi) if epi is not None else None
        L.mph_spmm_part(self.h, part, inp.data_ptr(), w, inp.stride(0), out.data_ptr(), out.stride(0), e,
                        stream_ptr(stream))
        return out

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            _destroy("mph_graph_destroy", h)
            self.h = None


class Features:
    """a1 — feature analysis + dense/sparse switch (Alg. 1 Initialize)."""

    def __init__(self, X: torch.Tensor, tau_bp: int = L.TAU_B200_BP, force_mode: int = -1, stream=None):
        assert X.is_cuda and X.dtype == torch.float32 and X.dim() == 2 and X.stride(1) == 1
        h = _out_ptr()
        L.mph_features_create(X.data_ptr(), X.shape[0], X.shape[1], X.stride(0), tau_bp, force_mode,
                              stream_ptr(stream), C.byref(h))
        self._attach(h, X.shape[0], X.shape[1])

    def _attach(self, h, N: int, F: int):
        self.h = h
        self.N, self.F = N, F
        nnz, mode, binary = C.c_int64(), C.c_int32(), C.c_int32()
        L.mph_features_info(h, C.byref(nnz), C.byref(mode), C.byref(binary))
        self.nnz, self.mode, self.is_binary = nnz.value, mode.value, bool(binary.value)

    @staticmethod
    def global_mode(nnz_local: int, n_local: int, F: int, tau_bp: int = L.TAU_B200_BP, pg=None) -> int:
        """The dense/sparse switch of a row-partitioned X (mph_features_decide on the global
        count): the per-rank nnz and row counts are summed over the torch.distributed group
        (plumbing); every rank gets the same mode to pass as force_mode."""
        import torch.distributed as dist
        t = torch.tensor([int(nnz_local), int(n_local)], dtype=torch.int64)
        if dist.is_initialized() and dist.get_world_size(pg) > 1:
            if dist.get_backend(pg) == "nccl":
                t = t.cuda()
            dist.all_reduce(t, group=pg)
        nnz, n = (int(v) for v in t.cpu().tolist())
        mode = C.c_int32()
        L.mph_features_decide(nnz, n, int(F), int(tau_bp), C.byref(mode))
        return mode.value

    @staticmethod
    def count_nnz(X: torch.Tensor, stream=None) -> int:
        """nnz of a device X (mph_features_count; synchronises)."""
        assert X.is_cuda and X.dtype == torch.float32 and X.dim() == 2 and X.stride(1) == 1
        n = C.c_int64()
        L.mph_features_count(X.data_ptr(), X.shape[0], X.shape[1], X.stride(0), stream_ptr(stream), C.byref(n))
        return n.value

    @classmethod
    def from_csr(cls, ptr: np.ndarray, idx: np.ndarray, val: np.ndarray, shape, tau_bp: int = L.TAU_B200_BP,
                 force_mode: int = -1, stream=None) -> "Features":
        """a1 from a host CSR matrix (mph_features_create_csr): NELL-sized X never densified."""
        p = np.ascontiguousarray(ptr, dtype=np.int64)
        i = np.ascontiguousarray(idx, dtype=np.int32)
        v = np.ascontiguousarray(val, dtype=np.float32)
        N, F = int(shape[0]), int(shape[1])
        assert p.shape == (N + 1,) and i.shape == v.shape
        h = _out_ptr()
        L.mph_features_create_csr(p.ctypes.data, i.ctypes.data, v.ctypes.data, N, F, tau_bp, force_mode,
                                  stream_ptr(stream), C.byref(h))
        self = cls.__new__(cls)
        self._attach(h, N, F)
        return self

    def csr(self):
        p, i, v = C.c_void_p(), C.c_void_p(), C.c_void_p()
        L.mph_features_csr(self.h, C.byref(p), C.byref(i), C.byref(v))
        return (device_view(p.value, (self.N + 1,), torch.int64), device_view(i.value, (self.nnz,), torch.int32),
                device_view(v.value, (self.nnz,), torch.float32))

    def csc(self):
        p, i, v = C.c_void_p(), C.c_void_p(), C.c_void_p()
        L.mph_features_csc(self.h, C.byref(p), C.byref(i), C.byref(v))
        return (device_view(p.value, (self.F + 1,), torch.int64), device_view(i.value, (self.nnz,), torch.int32),
                device_view(v.value, (self.nnz,), torch.float32))

    def dense(self) -> torch.Tensor:
        x, ld = C.c_void_p(), C.c_int32()
        L.mph_features_dense(self.h, C.byref(x), C.byref(ld))
        return device_view(x.value, (self.N, ld.value), torch.float32)

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            _destroy("mph_features_destroy", h)
            self.h = None


def partition_greedy(row_ptr: np.ndarray, world: int):
    """Alg. 4 Phase III (mph_partition_greedy): (part int32[N], load int64[world])."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    n = rp.size - 1
    part = np.empty(n, dtype=np.int32)
    load = np.empty(world, dtype=np.int64)
    L.mph_partition_greedy(rp.ctypes.data, n, world, part.ctypes.data, load.ctypes.data)
    return part, load


def partition_components(row_ptr: np.ndarray, col_idx: np.ndarray, world: int):
    """Alg. 4 Phase II (mph_partition_components): (part or None when connected, n_components)."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int32)
    n = rp.size - 1
    part = np.empty(n, dtype=np.int32)
    nc = C.c_int32()
    L.mph_partition_components(rp.ctypes.data, ci.ctypes.data, n, world, part.ctypes.data, C.byref(nc))
    return (part if nc.value > 1 else None), nc.value


def partition_hierarchical(row_ptr: np.ndarray, col_idx: np.ndarray, world: int):
    """Alg. 4 Phases II-III (mph_partition_hierarchical): (part, phase)."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int32)
    n = rp.size - 1
    part = np.empty(n, dtype=np.int32)
    ph = C.c_int32()
    L.mph_partition_hierarchical(rp.ctypes.data, ci.ctypes.data, n, world, part.ctypes.data, C.byref(ph))
    return part, ph.value


def relabel(part: np.ndarray, world: int):
    """mph_relabel: (new_id int64[N], bounds int64[world+1])."""
    pa = np.ascontiguousarray(part, dtype=np.int32)
    new_id = np.empty(pa.size, dtype=np.int64)
    bounds = np.empty(world + 1, dtype=np.int64)
    L.mph_relabel(pa.ctypes.data, pa.size, world, new_id.ctypes.data, bounds.ctypes.data)
    return new_id, bounds


def partition_stats(row_ptr: np.ndarray, col_idx: np.ndarray, part: np.ndarray, world: int) -> np.ndarray:
    """mph_partition_stats: int64[world, 4] = {owned, Σ d̃, distinct ghosts, cut entries}."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int32)
    pa = np.ascontiguousarray(part, dtype=np.int32)
    out = np.empty((world, 4), dtype=np.int64)
    L.mph_partition_stats(rp.ctypes.data, ci.ctypes.data, rp.size - 1, pa.ctypes.data, world, out.ctypes.data)
    return out


class Plan:
    """D1-D4 host plan of one rank (mph_plan_create)."""

    def __init__(self, row_ptr: np.ndarray, col_idx: np.ndarray, num_nodes: int, bounds: np.ndarray, rank: int):
        self._rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        self._ci = np.ascontiguousarray(col_idx, dtype=np.int32)
        self._b = np.ascontiguousarray(bounds, dtype=np.int64)
        self.world = len(self._b) - 1
        self.rank = rank
        h = _out_ptr()
        L.mph_plan_create(self._rp.ctypes.data, self._ci.ctypes.data, int(num_nodes), self._b.ctypes.data,
                          self.world, rank, C.byref(h))
        self.h = h
        n_own, row0, ng, nnz, ns = C.c_int32(), C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        L.mph_plan_info(h, C.byref(n_own), C.byref(row0), C.byref(ng), C.byref(nnz), C.byref(ns))
        self.n_own, self.row0, self.n_ghost, self.nnz, self.n_send = n_own.value, row0.value, ng.value, nnz.value, ns.value

    def arrays(self) -> dict:
        ptrs = [C.c_void_p() for _ in range(9)]
        L.mph_plan_arrays(self.h, *[C.byref(p) for p in ptrs])
        w = self.world

        def arr(p, n, ct, dt):
            if n == 0:
                return np.zeros(0, dtype=dt)
            return np.ctypeslib.as_array(C.cast(p, C.POINTER(ct)), shape=(n,)).copy()

        return {
            "ghosts": arr(ptrs[0].value, self.n_ghost, C.c_int64, np.int64),
            "row_ptr": arr(ptrs[1].value, self.n_own + 1, C.c_int64, np.int64),
            "col_idx": arr(ptrs[2].value, self.nnz, C.c_int32, np.int32),
            "split": arr(ptrs[3].value, self.n_own, C.c_int64, np.int64),
            "deg_local": arr(ptrs[4].value, self.n_own + self.n_ghost, C.c_int32, np.int32),
            "recv_offset": arr(ptrs[5].value, w, C.c_int64, np.int64),
            "n_recv": arr(ptrs[6].value, w, C.c_int64, np.int64),
            "send_offset": arr(ptrs[7].value, w + 1, C.c_int64, np.int64),
            "send_ids": arr(ptrs[8].value, self.n_send, C.c_int32, np.int32),
        }

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            _destroy("mph_plan_destroy", h)
            self.h = None


_ALLOC_T = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
_RELEASE_T = C.CFUNCTYPE(None, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
_torch_alloc_state = {}


def use_torch_allocator(on: bool = True) -> dict:
    """Route the library's internal device allocations through torch's caching allocator
    (mph_set_allocator); returns the live-allocation table {ptr: tensor} for inspection."""
    if not on:
        L.mph_set_allocator(None, None, None)
        return _torch_alloc_state.setdefault("live", {})
    live = _torch_alloc_state.setdefault("live", {})

    def alloc(nbytes, stream, ctx):
        t = torch.empty(int(nbytes), dtype=torch.uint8, device="cuda")
        live[t.data_ptr()] = t
        return t.data_ptr()

    def release(ptr, nbytes, stream, ctx):
        live.pop(int(ptr), None)

    cbs = (_ALLOC_T(alloc), _RELEASE_T(release))
    _torch_alloc_state["cbs"] = cbs   # the callbacks must outlive their registration
    L.mph_set_allocator(C.cast(cbs[0], C.c_void_p), C.cast(cbs[1], C.c_void_p), None)
    return live


def partition_1d(row_ptr: np.ndarray, world: int) -> np.ndarray:
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    out = np.zeros(world + 1, dtype=np.int64)
    L.mph_partition_1d(rp.ctypes.data, int(rp.size - 1), int(world), out.ctypes.data)
    return out


class Comm:
    """NCCL communicator; the unique id travels over torch.distributed (plumbing only)."""

    def __init__(self, world: int, rank: int, pg=None):
        import torch.distributed as dist
        buf = (C.c_uint8 * 128)()
        if rank == 0:
            L.mph_comm_unique_id(C.cast(buf, C.c_void_p))
        t = torch.tensor(list(bytes(buf)), dtype=torch.uint8)
        if dist.get_backend(pg) == "nccl":
            t = t.cuda()
        dist.broadcast(t, src=0, group=pg)
        ids = bytes(t.cpu().tolist())
        C.memmove(buf, ids, 128)
        h = _out_ptr()
        L.mph_comm_create(C.cast(buf, C.c_void_p), world, rank, C.byref(h))
        self.h = h
        self.world, self.rank = world, rank

    def allreduce_(self, t: torch.Tensor, stream=None):
        L.mph_allreduce_sum(self.h, t.data_ptr(), t.numel(), int(t.dtype == torch.float64), stream_ptr(stream))
        return t

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            _destroy("mph_comm_destroy", h)
            self.h = None


class GCN:
    """The L-layer GCN training step (initializeLayers / forwardPass / backPropagation / optimizer)."""

    def __init__(self, graph: Graph, features: Features, dims, dropout_p: float = 0.0, dropout_seed: int = 0,
                 order_policy: int = 0, comm: "Comm | str | None" = None, stream=None, aggregator: str = "gcn",
                 pg=None, precision: str = "tf32"):
        """comm: None (one GPU), a Comm (NCCL halo + all-reduce) or "p2p" (NVLink peer memory,
        NEXT-1): the ranks' arena descriptors are all-gathered over the torch.distributed group
        `pg` (plumbing only) and mapped by mph_gcn_p2p_open."""
        self.graph, self.features = graph, features
        p2p = isinstance(comm, str)
        if p2p and comm != "p2p":
            raise ValueError(f"comm must be a Comm, 'p2p' or None, not {comm!r}")
        self.comm = None if p2p else comm
        self.comm_mode = "p2p" if p2p else "nccl"
        self.dims = tuple(int(d) for d in dims)
        self.L = len(self.dims) - 1
        self.aggregator = aggregator
        arr = (C.c_int32 * len(self.dims))(*self.dims)
        self.precision = precision
        desc = GcnDesc(self.L, arr, float(dropout_p), int(dropout_seed), int(order_policy), L.AGG[aggregator],
                       L.COMM[self.comm_mode], L.PREC[precision])
        h = _out_ptr()
        L.mph_gcn_create(graph.h, features.h, C.byref(desc), self.comm.h if self.comm is not None else None,
                         stream_ptr(stream), C.byref(h))
        self.h = h
        if p2p:
            self._p2p_open(pg, stream)
        n = C.c_int64()
        offs = (C.c_int64 * (2 * self.L))()
        lds = (C.c_int32 * self.L)()
        L.mph_gcn_param_layout(h, C.byref(n), C.cast(offs, C.c_void_p), C.cast(lds, C.c_void_p))
        self.num_params = n.value
        self.offsets = list(offs)
        self.ld_w = list(lds)
        ptrs = [C.c_void_p() for _ in range(4)]
        L.mph_gcn_buffers(h, *[C.byref(p) for p in ptrs])
        self.params_flat, self.grads_flat, self.adam_m, self.adam_v = (
            device_view(p.value, (self.num_params,), torch.float32) for p in ptrs)
        order = (C.c_int32 * self.L)()
        mode = C.c_int32()
        L.mph_gcn_info(h, C.cast(order, C.c_void_p), C.byref(mode))
        self.order = list(order)
        self.loss_buf = torch.zeros(1, dtype=torch.float64, device="cuda")
        self._labels = None

    def _p2p_open(self, pg, stream):
        import torch.distributed as dist
        blob = (C.c_uint8 * L.P2P_BLOB_BYTES)()
        L.mph_gcn_p2p_export(self.h, C.cast(blob, C.c_void_p))
        world = dist.get_world_size(pg)
        mine = torch.tensor(list(bytes(blob)), dtype=torch.uint8)
        if dist.get_backend(pg) == "nccl":
            mine = mine.cuda()
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine, group=pg)
        allb = np.concatenate([p.cpu().numpy() for p in parts]).astype(np.uint8)
        L.mph_gcn_p2p_open(self.h, allb.ctypes.data, world, stream_ptr(stream))

    def p2p_status(self, detail: bool = False):
        """0, or MPH_ETIMEOUT (-10) when a peer-memory wait gave up (NEXT-1).  detail=True also
        returns the generation and the flag rows [4 slots][world] (halo, loss, grad, setup)."""
        e, gen = C.c_int32(), C.c_int64()
        world = max(1, self.graph_world())
        flags = np.zeros(4 * world, dtype=np.uint64)
        L.mph_gcn_p2p_status(self.h, C.byref(e), C.byref(gen), flags.ctypes.data)
        if detail:
            return e.value, gen.value, flags.reshape(4, world)
        return e.value

    def graph_world(self) -> int:
        return getattr(self.graph, "world", 1)

    # -- parameter views ([F_in][F_out] weights, [F_out] biases; padding excluded)
    def _views(self, flat):
        out = []
        for l in range(self.L):
            fin, fout = self.dims[l], self.dims[l + 1]
            ld = self.ld_w[l]
            W = flat[self.offsets[2 * l]:self.offsets[2 * l] + fin * ld].view(fin, ld)[:, :fout]
            b = flat[self.offsets[2 * l + 1]:self.offsets[2 * l + 1] + fout]
            out.append((W, b))
        return out

    def params(self):
        return self._views(self.params_flat)

    def grads(self):
        return self._views(self.grads_flat)

    def workspace_size(self) -> int:
        b = C.c_size_t()
        L.mph_gcn_workspace_size(self.h, C.byref(b))
        return b.value

    def bind(self, params=None, grads=None, adam_m=None, adam_v=None, workspace=None):
        """mph_gcn_bind: caller-owned (torch) buffers for the parameters, gradients, Adam moments
        and workspace; None keeps the model's own.  Refresh with params_updated()/init_xavier()."""
        def ptr(t, n_floats=None):
            if t is None:
                return None
            assert t.is_cuda and t.is_contiguous()
            if n_floats is not None:
                assert t.dtype == torch.float32 and t.numel() >= n_floats
            return t.data_ptr()
        ws_bytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
        L.mph_gcn_bind(self.h, ptr(params, self.num_params), ptr(grads, self.num_params), ptr(adam_m, self.num_params),
                       ptr(adam_v, self.num_params), ptr(workspace), ws_bytes)
        self._bound = (params, grads, adam_m, adam_v, workspace)   # keep alive
        ptrs = [C.c_void_p() for _ in range(4)]
        L.mph_gcn_buffers(self.h, *[C.byref(p) for p in ptrs])
        self.params_flat, self.grads_flat, self.adam_m, self.adam_v = (
            device_view(p.value, (self.num_params,), torch.float32) for p in ptrs)

    def init_xavier(self, seed: int = 42, stream=None):
        L.mph_gcn_init_xavier(self.h, int(seed), stream_ptr(stream))

    def params_updated(self, stream=None):
        L.mph_gcn_params_updated(self.h, stream_ptr(stream))

    def set_labels(self, labels: torch.Tensor, mask: torch.Tensor | None = None, n_lab_global: int | None = None):
        assert labels.is_cuda and labels.dtype == torch.int32
        if mask is not None:
            assert mask.is_cuda and mask.dtype == torch.uint8
        if n_lab_global is None:
            n_lab_global = int(mask.sum().item()) if mask is not None else labels.numel()
            if self.graph_world() > 1:
                # the loss is a mean over the GLOBAL labelled rows: sum the local counts
                import torch.distributed as dist
                if not dist.is_initialized():
                    raise ValueError("set_labels on a partitioned graph needs n_lab_global "
                                     "(or an initialised torch.distributed group to sum the counts)")
                t = torch.tensor([n_lab_global], dtype=torch.int64)
                if dist.get_backend() == "nccl":
                    t = t.cuda()
                dist.all_reduce(t)
                n_lab_global = int(t.item())
        self._labels = (labels, mask)  # keep alive
        L.mph_gcn_set_labels(self.h, labels.data_ptr(), mask.data_ptr() if mask is not None else None,
                             int(n_lab_global))

    def forward(self, epoch: int = 1, stream=None):
        L.mph_gcn_forward(self.h, int(epoch), stream_ptr(stream))

    def loss(self, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        out = self.loss_buf if out is None else out
        L.mph_gcn_loss(self.h, out.data_ptr(), stream_ptr(stream))
        return out

    def backward(self, stream=None):
        L.mph_gcn_backward(self.h, stream_ptr(stream))

    def adam(self, t: int, cfg=DEFAULT_ADAM, stream=None):
        L.mph_gcn_adam(self.h, C.byref(AdamCfg(*cfg)), int(t), stream_ptr(stream))

    def optim_step(self, t: int, cfg: OptimCfg, stream=None):
        L.mph_gcn_optim_step(self.h, C.byref(cfg), int(t), stream_ptr(stream))

    def train_epoch(self, t: int, cfg=DEFAULT_ADAM, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """cfg: an Adam tuple (lr, b1, b2, eps) or an OptimCfg from optimizer(...)."""
        out = self.loss_buf if out is None else out
        if isinstance(cfg, OptimCfg):
            L.mph_gcn_train_epoch_opt(self.h, int(t), C.byref(cfg), out.data_ptr(), stream_ptr(stream))
        else:
            L.mph_gcn_train_epoch(self.h, int(t), C.byref(AdamCfg(*cfg)), out.data_ptr(), stream_ptr(stream))
        return out

    def graph_capture(self, t_next: int, cfg=DEFAULT_ADAM, stream=None):
        """Record one whole epoch as a CUDA graph; each replay() then runs the next epoch."""
        if isinstance(cfg, OptimCfg):
            L.mph_gcn_graph_capture_opt(self.h, C.byref(cfg), int(t_next), stream_ptr(stream))
        else:
            L.mph_gcn_graph_capture(self.h, C.byref(AdamCfg(*cfg)), int(t_next), stream_ptr(stream))
        t, loss = C.c_void_p(), C.c_void_p()
        L.mph_gcn_graph_state(self.h, C.byref(t), C.byref(loss))
        self.graph_step = device_view(t.value, (1,), torch.int32)
        self.graph_loss = device_view(loss.value, (1,), torch.float64)

    def replay(self, stream=None) -> torch.Tensor:
        L.mph_gcn_graph_replay(self.h, stream_ptr(stream))
        return self.graph_loss

    def tensor(self, kind: int, layer: int) -> torch.Tensor:
        """Borrowed view of an activation (mph_gcn_tensor): float32, or bfloat16 for the GEMM-only
        tensors of a BF16-precision model."""
        p, rows, width, ld, eb = C.c_void_p(), C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        L.mph_gcn_tensor(self.h, kind, layer, C.byref(p), C.byref(rows), C.byref(width), C.byref(ld), C.byref(eb))
        if not p.value:
            return None
        if eb.value == 2:
            raw = device_view(p.value, (rows.value, ld.value), torch.int16)
            return raw.view(torch.bfloat16)[:, :width.value]
        return device_view(p.value, (rows.value, ld.value), torch.float32)[:, :width.value]

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            _destroy("mph_gcn_destroy", h)
            self.h = None
