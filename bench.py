#!/usr/bin/env python
"""Benchmark: GCN ms/epoch (fwd+bwd+Adam) on B200, with SpMM roofline and CPU-oracle baseline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config reddit] [--impl ours|reference]

One JSON line on rank 0 (BASELINE.json metric).  An epoch is SURVEY §8(d)'s step a2..a11:
forward, softmax-CE, backward, (halo + gradient all-reduce when N > 1) and Adam, on a
synthetic graph shaped like the named config (synth/, seeded).  For N > 1 launch with
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P bench.py --gpus N
(one rank per GPU; the graph is 1D row-partitioned, so total work is fixed: strong scaling).  The
halo rows and the gradient sum travel over NVLink peer memory by default (--comm p2p, SURVEY §8(f)
NEXT-1: the ranks map each other's buffers via CUDA IPC; torch.distributed only all-gathers the
descriptors, barriers and takes the max of the timings) or through NCCL (--comm nccl).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "GCN ms/epoch (fwd+bwd+Adam) at 1/2/4/8 B200; SpMM HBM GB/s vs peak"
UNIT = "ms/epoch"
FALLBACK_HBM_GBS = 6650.0
PROF_KINDS = {0: "spmm", 1: "gemm_nt", 2: "gemm_tn", 3: "softmax_ce", 4: "adam", 5: "sparse_feat", 6: "halo"}


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:   # driver-written; tolerate {"hbm_gbs": 7100.0} or {"hbm_gbs": {"value": 7100.0, ...}}
            with open(p) as f:
                v = json.load(f).get("hbm_gbs")
            if isinstance(v, dict):
                v = v.get("value", v.get("gbs", v.get("burst")))
            if v is not None and float(v) > 0:
                return float(v), "measured"
        except (OSError, ValueError, TypeError, AttributeError):
            pass
    return FALLBACK_HBM_GBS, "fallback"


# ---------------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------------- CPU oracle
def _oracle_inputs(w):
    """The oracle's view of the SAME workload the GPU arm trains (full size, no scaling): its own
    CSR build (setup, untimed) and the cached Â operator."""
    import oracle
    cfg = w["cfg"]
    g = oracle.graph_build(w["src"], w["dst"], cfg.num_nodes)
    oracle.prepare(g)
    if w.get("X") is not None:
        X = w["X"]
    else:
        import scipy.sparse as sp
        ptr, idx, val = w["X_csr"]
        X = sp.csr_matrix((val, idx, ptr), shape=(cfg.num_nodes, cfg.num_features))
    return g, X


def _oracle_epochs_ms(w, g, X, epochs: int):
    """Time `epochs` full epochs of the oracle as it stands (forward, softmax-CE, backward, Adam on
    the whole graph, Listing 1) on the full workload; per-epoch wall ms."""
    import oracle
    cfg = w["cfg"]
    dims = cfg.dims
    Ws, bs = oracle.xavier_init(dims, 42)
    params = [np.asarray(a, np.float64).copy() for a in Ws] + [np.asarray(b, np.float64).copy() for b in bs]
    L_ = len(Ws)
    m = [np.zeros_like(p) for p in params]
    v = [np.zeros_like(p) for p in params]
    times = []
    for t in range(1, epochs + 1):
        t0 = time.perf_counter()
        Z, cache = oracle.forward(g, X, params[:L_], params[L_:], epoch=t)
        _, dZ = oracle.softmax_ce(Z, w["y"])
        dW, db = oracle.backward(g, cache, params[:L_], dZ)
        oracle.adam_step(params, dW + db, m, v, t)
        times.append((time.perf_counter() - t0) * 1e3)
        del Z, cache, dZ
    return times


def _cpu_threads():
    """Threads the oracle actually uses: its row-parallel sparse products (oracle.threads_used)
    and the BLAS pool of its dense products (threadpoolctl)."""
    import oracle
    blas = 1
    try:
        from threadpoolctl import threadpool_info
        blas = max((int(i.get("num_threads", 1)) for i in threadpool_info()), default=1)
    except Exception:
        pass
    return max(oracle.threads_used(), blas), {"sparse_products": oracle.threads_used(), "blas": blas,
                                             "host_cpus": os.cpu_count()}


def _sample_desc(w, epochs):
    c = w["cfg"]
    return (f"oracle (FP64 numpy/scipy, row-parallel sparse products) on the full {c.name}-shaped workload "
            f"(N={c.num_nodes}, nnz(A)={c.nnz_a}, dims={list(c.dims)}): {epochs} whole epoch(s) "
            f"(forward + softmax-CE + backward + Adam), no scaling")


def _config_common(args, world):
    """The config keys both arms report (the reference arm adds how the oracle sampled it)."""
    from synth.generate import CONFIGS
    cfg = CONFIGS[args.config]
    return {"workload": args.config, "nodes": cfg.num_nodes, "nnz_A": cfg.nnz_a, "dims": list(cfg.dims),
            "layers": cfg.num_layers, "global_batch": cfg.num_nodes, "seq_len": None,
            "parallelism": (f"1d-row-partition x{world}" + ("" if args.partition == "1d" else
                                                             f" ({args.partition} + relabel)") + f", comm {args.comm}")
            if world > 1 else "single-gpu"}


def run_reference(args):
    """The reference arm of this tier is the oracle (task ③/④): the SAME full-size workload as our
    arm, each step one whole oracle epoch, W warm-up + K timed steps on the host cores."""
    rank = _env_int("RANK", 0)
    if rank != 0:
        return 0
    from synth.generate import make_workload
    w = make_workload(args.config)
    g, X = _oracle_inputs(w)
    ms_all = _oracle_epochs_ms(w, g, X, args.warmup + args.steps)
    ms = ms_all[args.warmup:]
    v = statistics.median(ms)
    cores, detail = _cpu_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": v, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {**_config_common(args, args.gpus), "oracle_scale": "1/1 (full size)"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "threads": detail, "kind": "oracle",
                         "sample": _sample_desc(w, args.steps)},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "epoch_ms": {"median": v, "min": min(ms), "max": max(ms), "timed_region_s": sum(ms) / 1e3},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------- our arm
def _relabel_workload(P, torch, w, world, how):
    """Alg. 4 partition (NEXT-3) + relabelling: returns the workload in new ids and the contiguous
    bounds that realise the partition.  Host work, outside the timed region."""
    n = w["cfg"].num_nodes
    g = P.Graph(w["src"], w["dst"], n)
    rp, ci = (t.cpu().numpy() for t in g.csr()[:2])
    del g
    part = P.partition_greedy(rp, world)[0] if how == "greedy" else P.partition_hierarchical(rp, ci, world)[0]
    new_id, bounds = P.relabel(part, world)
    inv = np.empty(n, dtype=np.int64)
    inv[new_id] = np.arange(n)
    out = dict(w, src=new_id[w["src"]].astype(np.int32), dst=new_id[w["dst"]].astype(np.int32), y=w["y"][inv])
    if w["X"] is not None:
        out["X"] = np.ascontiguousarray(w["X"][inv])
    else:
        ptr, idx, val = w["X_csr"]
        lens = np.diff(ptr)[inv]
        nptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(lens, out=nptr[1:])
        take = np.concatenate([np.arange(ptr[v], ptr[v + 1]) for v in inv]) if n else np.zeros(0, np.int64)
        out["X_csr"] = (nptr, idx[take], val[take])
    return out, bounds


def _build_model(P, torch, w, world, rank, comm, bounds=None, precision="tf32", aggregator="gcn"):
    cfg = w["cfg"]
    n = cfg.num_nodes
    X = w["X"]

    def features(r0, r1):
        # the dense/sparse switch is decided on the GLOBAL nonzero count (identical on every rank)
        if X is not None:
            Xd = torch.from_numpy(np.ascontiguousarray(X[r0:r1])).cuda()
            mode = P.Features.global_mode(P.Features.count_nnz(Xd), r1 - r0, cfg.num_features) if world > 1 else -1
            return P.Features(Xd, force_mode=mode)
        ptr, idx, val = w["X_csr"]   # CSR features (NELL): rows r0..r1 of the host CSR, never densified
        b, e = int(ptr[r0]), int(ptr[r1])
        mode = P.Features.global_mode(e - b, r1 - r0, cfg.num_features) if world > 1 else -1
        return P.Features.from_csr(ptr[r0:r1 + 1] - b, idx[b:e], val[b:e], (r1 - r0, cfg.num_features),
                                   force_mode=mode)

    if world == 1:
        g = P.Graph(w["src"], w["dst"], n)
        f = features(0, n)
        m = P.GCN(g, f, cfg.dims, precision=precision, aggregator=aggregator)
        y = torch.from_numpy(w["y"]).cuda()
        own = (0, n)
        extra = {}
    else:
        gfull = P.Graph(w["src"], w["dst"], n)
        rp, ci = gfull.csr()[0].cpu().numpy(), gfull.csr()[1].cpu().numpy()
        del gfull
        if bounds is None:
            bounds = P.partition_1d(rp, world)
        plan = P.Plan(rp, ci, n, bounds, rank)
        del rp, ci
        g = P.Graph.from_plan(plan)
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        f = features(r0, r1)
        m = P.GCN(g, f, cfg.dims, comm=comm, precision=precision, aggregator=aggregator)
        y = torch.from_numpy(np.ascontiguousarray(w["y"][r0:r1])).cuda()
        own = (r0, r1)
        extra = {"n_ghost": plan.n_ghost, "halo_rows_sent": plan.n_send}
    m.init_xavier(42)
    m.set_labels(y, n_lab_global=n)
    return g, f, m, y, own, extra


def _spmm_widths(P, m):
    """Padded widths of one epoch's aggregation calls (forward, then backward), from the layer
    orders of reading Q7: a transform-first layer aggregates its output width forward and
    backward; an aggregate-first layer 1 aggregates its input width forward only."""
    dims = m.dims
    fwd, bwd = [], []
    for l, o in enumerate(m.order):
        if o == 1:
            fwd.append(P.pad_width(dims[l]))
        else:
            fwd.append(P.pad_width(dims[l + 1]))
            bwd.append(P.pad_width(dims[l + 1]))
    return fwd + bwd[::-1]


def _spmm_fractions(r, peak_hbm, l2_gather_gbps, l2_bytes=126 * 2 ** 20):
    """SURVEY §8(d) d.4's three SpMM roofline fractions for one measured workload: (1) ncu DRAM
    bytes / time / HBM peak, (2) time efficiency E = T_floor / T_measured with T_floor =
    Σ_calls max(floor bytes / HBM, [operand <= L2] · nnz·4·w / L2-gather), (3) algorithmic
    (no-reuse) bytes / time / HBM peak (== roofline.frac)."""
    k = r["kernels"].get("spmm")
    geo = r.get("_spmm_geometry")
    if not k or not geo:
        return None
    n, nc, nnz = geo["n_rows"], geo["n_cols"], geo["nnz"]
    t_floor_ms = 0.0
    for wpad in geo["widths"]:
        floor_bytes = 4.0 * wpad * (nc + n) + 4.0 * nnz + 8.0 * (n + 1) + 4.0 * n
        t = floor_bytes / (peak_hbm * 1e6)
        if l2_gather_gbps and nc * 4.0 * wpad <= l2_bytes:
            t = max(t, nnz * 4.0 * wpad / (l2_gather_gbps * 1e6))
        t_floor_ms += t
    out = {"time_efficiency_E": t_floor_ms / k["ms_per_epoch"], "floor_ms_per_epoch": t_floor_ms,
           "widths": geo["widths"], "effective_frac_of_hbm": k["algorithmic_GBps"] / peak_hbm,
           "l2_gather_GBps_used": l2_gather_gbps}
    traffic = (r.get("roofline") or {}).get("traffic")
    if traffic:
        out["dram_frac_of_hbm"] = traffic / (k["avg_launch_ms"] * 1e6) / peak_hbm
    return out


PEAKS = {}   # filled by run_ours before any workload is timed (probes + MEASURED_PEAKS.json)


def _l2_ceiling(peaks):
    """(GB/s, source) of the L2 delivery ceiling: the LTS byte peak ncu reports for this part
    (profiles/l2_peak.json: lts__t_bytes.sum.peak_sustained x the L2 clock, 34.6 TB/s on B200), a
    rate no kernel can exceed; without that file, the best of this run's probes (an L2-resident
    streaming read and random-row gather), which the aggregation itself can beat."""
    p = os.path.join(ROOT, "profiles", "l2_peak.json")
    if os.path.exists(p):
        try:
            with open(p) as f:
                v = float(json.load(f)["lts_bytes_peak_GBps"])
            return v, ("ncu LTS byte peak of B200 (lts__t_bytes.sum.peak_sustained x L2 clock = "
                       f"{v:.0f} GB/s, profiles/l2_peak.json)")
        except (OSError, ValueError, KeyError, TypeError):
            pass
    cands = [peaks.get("l2_stream_GBps"), (peaks.get("gather") or {}).get("l2_resident_64MB")]
    cands = [c for c in cands if c]
    if not cands:
        return None, None
    return max(cands), "measured in this run: max(L2 streaming-read probe, L2-resident random-row gather probe)"


def _roofline(kernels, ms, config, peaks):
    """Roofline of the epoch's dominant kernel (task ④).

    Aggregation SpMM: achieved = SURVEY §8(d) d.3's per-edge algorithmic bytes (4 B id + 4·w B
    gathered row, the no-reuse amount Alg. 3 reads) plus per-row bytes, x the launch's
    edges, / its CUDA-event launch time.  Every one of those bytes is delivered to the SMs by L2
    (or hits L1), so the ceiling is the L2 delivery rate measured in this run (bound "l2"), not
    HBM: DRAM only sees the misses (`traffic`, from the ncu capture of this code).  The
    north star's literal "SpMM HBM GB/s vs peak" is dram_frac_of_hbm = traffic / time / HBM peak.
    Other kernels: algorithmic bytes (A + B + C once) / time against the HBM copy peak."""
    hbm, hbm_kind = peaks.get("hbm_gbs"), peaks.get("hbm_kind")
    dom = max((k for k in ("spmm", "gemm_nt", "gemm_tn", "sparse_feat") if k in kernels),
              key=lambda k: kernels[k]["ms_per_epoch"], default=None)
    if dom is None:
        return None
    kd = kernels[dom]
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"ncu_traffic_{config}.json")
    if os.path.exists(tp):
        with open(tp) as fh:
            traffic = json.load(fh).get(dom, {}).get("dram_bytes_per_launch")
    hbm_src = ("MEASURED_PEAKS.json hbm_gbs (of measured)" if hbm_kind == "measured" else
               "fallback 6.65 TB/s of B200_PROFILING.md (MEASURED_PEAKS.json absent)")
    l2, l2_src = _l2_ceiling(peaks)
    gathering = dom in ("spmm", "sparse_feat")
    if gathering and l2:
        r = {"bound": "l2", "kernel": dom, "achieved": kd["algorithmic_GBps"], "peak": l2, "unit": "GB/s",
             "frac": kd["algorithmic_GBps"] / l2, "traffic": traffic,
             "peak_source": l2_src + "; every gathered byte reaches the SMs through L2 (or hits L1), DRAM only "
                                     "sees the misses (traffic)"}
    else:
        r = {"bound": "hbm", "kernel": dom, "achieved": kd["algorithmic_GBps"], "peak": hbm, "unit": "GB/s",
             "frac": kd["algorithmic_GBps"] / hbm, "traffic": traffic, "peak_source": hbm_src}
    r["algorithmic_bytes"] = ("SURVEY 8(d) d.3 per edge of A-hat 4 + 4*w_pad B (id + gathered row, no reuse), "
                              "per row 12 + 4*w_pad B" if dom == "spmm" else
                              "per nonzero of X 8 + 4*w B, per row/column 8 + 4*w B" if dom == "sparse_feat" else
                              "A + B + C bytes once")
    r.update({"bytes_per_launch": kd["bytes_per_launch"], "avg_launch_ms": kd["avg_launch_ms"],
              "share_of_epoch": kd["ms_per_epoch"] / ms, "hbm_peak": hbm, "hbm_peak_source": hbm_src})
    if traffic:
        r["dram_frac_of_hbm"] = traffic / (kd["avg_launch_ms"] * 1e6) / hbm
        r["traffic_source"] = f"profiles/ncu_traffic_{config}.json (ncu --set full of this code, per launch)"
    if "halo" in kernels:   # SURVEY d.4: halo bytes per rank / time / NVLink (measured peer copy, 770 GB/s)
        r["halo_frac_of_nvlink_peer_copy_770GBps"] = kernels["halo"]["algorithmic_GBps"] / 770.0
    return r


def _max_over_ranks(torch, dist, v: float) -> float:
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    tt = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    return tt.item()


_WORKLOADS = {}


def _measure(P, L, torch, dist, C, args, config, world, rank, local, comm, full: bool):
    """Build one workload and time it.  full=False skips e2e and the CPU baseline (secondary)."""
    t_setup = time.perf_counter()
    from synth.generate import make_workload
    if config not in _WORKLOADS:   # one generation per config per run (secondary lines reuse it)
        _WORKLOADS.clear()
        _WORKLOADS[config] = make_workload(config)
    w = _WORKLOADS[config]
    t_gen = time.perf_counter() - t_setup
    t0 = time.perf_counter()
    bounds = None
    if world > 1 and args.partition != "1d":
        w, bounds = _relabel_workload(P, torch, w, world, args.partition)
    g, f, m, y, own, extra = _build_model(P, torch, w, world, rank, comm, bounds, args.precision, args.aggregator)
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    cfg = w["cfg"]
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    for t in range(1, args.warmup + 1):
        m.train_epoch(t)
    torch.cuda.synchronize()
    barrier()

    # ---------------- device-timed region: K epochs, inputs resident in HBM
    use_graph = bool(args.graph) and (world == 1 or args.comm == "p2p")
    if use_graph:  # one captured epoch, replayed K times (the per-kernel breakdown needs eager launches)
        m.graph_capture(args.warmup + 1)
    clocks = ClockSampler(local)
    L.mph_profile_enable(0 if use_graph else 1)
    launches0 = L.launch_count()
    clocks.start()
    time.sleep(0.15)
    barrier()
    torch.cuda.synchronize()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]   # one per epoch boundary
    evs[0].record(stream)
    for i, t in enumerate(range(args.warmup + 1, args.warmup + args.steps + 1)):
        if use_graph:
            m.replay()
        else:
            m.train_epoch(t)
        evs[i + 1].record(stream)
    ev0, ev1 = evs[0], evs[-1]
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    launches = L.launch_count() - launches0
    ms = ev0.elapsed_time(ev1) / args.steps
    per_epoch = sorted(evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps))
    q = lambda f: per_epoch[min(len(per_epoch) - 1, int(round(f * (len(per_epoch) - 1))))]  # noqa: E731
    epoch_stats = {"median": q(0.5), "p10": q(0.1), "p90": q(0.9), "unit": "ms", "this_rank": True}
    kernels = {}
    for kind, name in PROF_KINDS.items():
        cnt, tms, by, fl = C.c_int64(), C.c_double(), C.c_double(), C.c_double()
        L.mph_profile_read(kind, C.byref(cnt), C.byref(tms), C.byref(by), C.byref(fl))
        if cnt.value:
            kernels[name] = {"launches_per_epoch": cnt.value / args.steps, "ms_per_epoch": tms.value / args.steps,
                             "avg_launch_ms": tms.value / cnt.value, "algorithmic_GBps": by.value / tms.value / 1e6,
                             "bytes_per_launch": by.value / cnt.value, "TFLOPs": fl.value / tms.value / 1e9}
    L.mph_profile_enable(0)
    if "gemm_tn" in kernels:
        # gcn.cu: the weight-gradient GEMMs leave the critical path for a side stream when every
        # aggregation operand fits 512 MB (reddit, arxiv); their event span then includes the
        # concurrent aggregation, so it is wall time on that stream, not kernel time
        nc = w["cfg"].num_nodes
        side = nc * max(P.pad_width(d) for d in w["cfg"].dims[1:]) * 4.0 <= 512.0 * (1 << 20)
        kernels["gemm_tn"]["stream"] = ("side stream, overlapped with the next aggregation: ms is wall time on "
                                        "that stream, not kernel time") if side else "compute stream (in line)"
    loss_last = m.loss_buf.item()
    if world > 1 and args.comm == "p2p" and m.p2p_status() != 0:
        raise RuntimeError(f"rank {rank}: a peer-memory wait timed out (MPH_ETIMEOUT); the timings are invalid")
    if world > 1:
        ms = _max_over_ranks(torch, dist, ms)
        # evidence of the transport: which GPUs reach each other, whether any peer
        # wait timed out, and what one halo exchange moved and took on this rank
        ndev = torch.cuda.device_count()
        hk = kernels.get("halo")
        extra["transport"] = {
            "comm": args.comm,
            "peer_access": [[bool(i == j or torch.cuda.can_device_access_peer(i, j)) for j in range(ndev)]
                            for i in range(ndev)],
            "p2p_status": m.p2p_status() if args.comm == "p2p" else None,
            "halo_exchanges_per_epoch": hk["launches_per_epoch"] if hk else None,
            "halo_bytes_per_exchange": hk["bytes_per_launch"] if hk else None,
            "halo_ms_per_exchange": hk["avg_launch_ms"] if hk else None,
            "halo_GBps": hk["algorithmic_GBps"] if hk else None,
        }

    # ---------------- end-to-end through the public API with host buffers
    e2e = None
    if full and not args.no_e2e:
        upload = f.mode == 0   # sparse-mode features are analysed once at load (Alg. 1); labels still move
        if upload:
            X = w["X"][own[0]:own[1]]
            Pw = P.pad_width(X.shape[1])
            Xh = torch.zeros((X.shape[0], Pw), dtype=torch.float32).pin_memory()   # padded pinned host rows
            Xh[:, :X.shape[1]] = torch.from_numpy(X)
        else:
            Xh, Pw = torch.zeros(0), 0
        yh = torch.from_numpy(np.ascontiguousarray(w["y"][own[0]:own[1]])).pin_memory()
        lh = torch.zeros(1, dtype=torch.float64).pin_memory()
        steps_e2e = max(3, args.steps // 2)
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        copy_stream = torch.cuda.Stream()
        y_bufs = [y, torch.empty_like(y)]   # double-buffered labels: step i+1's land while step i reads

        def load_inputs(i):   # step i's inputs from pinned host memory, all H2D on the copy stream
            with torch.cuda.stream(copy_stream):
                y_bufs[i % 2].copy_(yh, non_blocking=True)   # epoch i-2, its last reader, has finished
            if upload:   # waits for the previous X to be consumed, copies, then the compute stream waits
                L.mph_gcn_upload_features_async(m.h, Xh.data_ptr(), Pw, copy_stream.cuda_stream, stream.cuda_stream)
            else:
                stream.wait_stream(copy_stream)

        d2h_stream = torch.cuda.Stream()
        e0.record(stream)
        base = args.warmup + args.steps
        load_inputs(0)
        for i, t in enumerate(range(base + 1, base + steps_e2e + 1)):
            m.set_labels(y_bufs[i % 2], n_lab_global=cfg.num_nodes)
            m.train_epoch(t)
            epoch_done = torch.cuda.Event()
            epoch_done.record(stream)
            if i + 1 < steps_e2e:
                load_inputs(i + 1)    # prefetch: the next step's copies overlap this epoch
            # the loss read-back is issued after the prefetch (the copy engines serve submissions in
            # order, so a D2H queued behind a running epoch would hold the next H2D back)
            d2h_stream.wait_event(epoch_done)
            with torch.cuda.stream(d2h_stream):
                lh.copy_(m.loss_buf, non_blocking=True)
            done = torch.cuda.Event()
            done.record(d2h_stream)
            done.synchronize()   # the step's result is on the host
        stream.wait_stream(d2h_stream)
        e1.record(stream)
        m.set_labels(y, n_lab_global=cfg.num_nodes)
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1) / steps_e2e
        if world > 1:
            e2e_ms = _max_over_ranks(torch, dist, e2e_ms)
        e2e = {"value": e2e_ms, "unit": UNIT, "h2d_bytes_per_step": int(Xh.numel() * 4 * upload + yh.numel() * 4),
               "d2h_bytes_per_step": 8, "steps": steps_e2e,
               "inputs": "features (padded, pinned) + labels H2D and loss D2H every step; the next step's "
                         "feature copy is issued on a copy stream while the current epoch runs (prefetch), the "
                         "host waits for each step's loss"}

    # ---------------- roofline of the dominant kernel
    roofline = _roofline(kernels, ms, config, PEAKS)
    # ---------------- CPU oracle baseline (rank 0, N = 1 only)
    cpu = None
    if full and world == 1 and rank == 0 and not args.no_cpu_baseline:
        og, oX = _oracle_inputs(w)
        ms_cpu = _oracle_epochs_ms(w, og, oX, 1)
        del og, oX
        cores, detail = _cpu_threads()
        cpu = {"value": statistics.median(ms_cpu), "unit": UNIT, "cores": cores, "threads": detail, "kind": "oracle",
               "sample": _sample_desc(w, 1)}

    out = {
        "value": ms, "ms_per_step": ms,
        "config": {**_config_common(argparse.Namespace(**{**vars(args), "config": config}), world),
                   "layer_order": ["AF" if o else "TF" for o in m.order],
                   "gemm_precision": args.precision,
                   "aggregator": args.aggregator,
                   "cuda_graph": use_graph,
                   "l2": "inputs larger than L2 (X and col_idx > 126 MB); no flush" if cfg.num_nodes > 100000
                   else "small workload: operands L2-resident across epochs (no flush)",
                   **extra},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk,
        "kernels": kernels, "final_loss": loss_last, "epoch_ms": epoch_stats,
        "_spmm_geometry": {"widths": _spmm_widths(P, m), "n_rows": g.n_rows,
                           "n_cols": g.n_cols, "nnz": g.nnz},
        "setup_s": {"generate": round(t_gen, 2), "graph_build_and_init": round(t_build, 2)},
    }
    del m, f, g
    return out


def _gather_peaks(L, torch):
    """Measured random-row gather bandwidth (512 B rows) from an L2-resident (64 MB) and an
    HBM-resident (4 GB) table: the ceilings the aggregation SpMM actually runs against."""
    res = {}
    w = 128
    out = torch.empty(148 * 32 * 128, device="cuda")
    n_idx = 1 << 24
    for name, table_bytes in (("l2_resident_64MB", 64 << 20), ("hbm_resident_4GB", 4 << 30)):
        rows = table_bytes // (w * 4)
        table = torch.ones((rows, w), device="cuda")
        idx = torch.randint(0, rows, (n_idx,), device="cuda", dtype=torch.int32)
        s = torch.cuda.current_stream()
        best = None
        for _ in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            L.mph_probe_gather(table.data_ptr(), rows, w, idx.data_ptr(), n_idx, out.data_ptr(), s.cuda_stream)
            e1.record(s)
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1)
            best = t if best is None else min(best, t)
        res[name] = n_idx * w * 4 / best / 1e6
        del table, idx
    torch.cuda.empty_cache()
    return res


def _l2_stream_peak(L, torch):
    """L2 delivery ceiling: streaming reads (no L1) of a ~50 MB L2-resident buffer, best of 5."""
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    unit = 8 * sms
    n = (50 << 20) // 4 // unit * unit
    buf = torch.ones(n, device="cuda")
    out = torch.empty(2 * sms * 512 * 4, device="cuda")
    s = torch.cuda.current_stream()
    passes, best = 20, None
    L.mph_probe_l2_stream(buf.data_ptr(), n, 2, out.data_ptr(), s.cuda_stream)   # warm: buffer into L2
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        L.mph_probe_l2_stream(buf.data_ptr(), n, passes, out.data_ptr(), s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
        best = t if best is None else min(best, t)
    del buf, out
    torch.cuda.empty_cache()
    return passes * n * 4 / best / 1e6


def run_ours(args):
    import ctypes as C

    import torch
    import torch.distributed as dist

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE", file=sys.stderr)
    if args.share_device:
        # functional check of the N > 1 code path on a one-GPU box: every rank on cuda:0, gloo
        # plumbing, P2P transport (ranks time-slice the GPU, so the timings mean nothing)
        if args.comm != "p2p":
            print("--share-device needs --comm p2p (NCCL refuses two ranks on one device)", file=sys.stderr)
            return 2
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if args.share_device:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2512_01678_b200 as P
    from paper_2512_01678_b200 import _lib as L

    L.mph_device_check(C.byref(C.c_int32()))
    if world > 1 and args.comm == "p2p" and not args.share_device:
        # peer memory needs every pair of the job's GPUs to reach each other (NVLink/NVSwitch); on a
        # box without peer access the halo and gradient sum go through NCCL instead (said in config)
        ok = all(torch.cuda.can_device_access_peer(local, d) for d in range(world) if d != local)
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device="cuda")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if not int(flag.item()):
            if rank == 0:
                print("no peer access between the GPUs: --comm nccl", file=sys.stderr)
            args.comm = "nccl"
    # N > 1: NCCL halo/all-reduce, or NVLink peer memory (NEXT-1: the model maps its peers itself)
    comm = (P.Comm(world, rank) if args.comm == "nccl" else "p2p") if world > 1 else None
    hbm, hbm_kind = _peaks()
    PEAKS.update({"hbm_gbs": hbm, "hbm_kind": hbm_kind})
    if not args.no_probe:   # measured before any workload: the ceilings the roofline divides by
        PEAKS["gather"] = _gather_peaks(L, torch)
        PEAKS["l2_stream_GBps"] = _l2_stream_peak(L, torch)
    main = _measure(P, L, torch, dist, C, args, args.config, world, rank, local, comm, full=True)
    secondary = {}
    for spec in ([] if args.secondary == "none" else args.secondary.split(",")):
        cfgname, _, prec = spec.partition(":")   # "products" or "reddit:bf16" (GEMM operand precision)
        prec = prec or args.precision
        if cfgname and (cfgname != args.config or prec != args.precision):
            sargs = argparse.Namespace(**{**vars(args), "precision": prec})
            r = _measure(P, L, torch, dist, C, sargs, cfgname, world, rank, local, comm, full=False)
            secondary[spec] = {k: r[k] for k in ("value", "config", "roofline", "kernels", "gpu_launches",
                                                 "final_loss", "clocks", "epoch_ms", "_spmm_geometry")}
    l2g = (PEAKS.get("gather") or {}).get("l2_resident_64MB")   # d.4's E: the L2 random-row gather rate
    l2_bytes = int(getattr(torch.cuda.get_device_properties(local), "L2_cache_size", 126 * 2 ** 20))
    for r in [main] + list(secondary.values()):
        if r.get("roofline") is not None:
            fr = _spmm_fractions(r, hbm, l2g, l2_bytes)
            if fr:
                r["roofline"]["spmm_fractions"] = fr
            if PEAKS.get("gather"):
                r["roofline"]["measured_probe_GBps"] = {**PEAKS["gather"], "l2_stream": PEAKS.get("l2_stream_GBps")}
        r.pop("_spmm_geometry", None)

    if rank == 0:
        line = {
            "metric": METRIC, "value": main["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": main["ms_per_step"], "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": f"f32 (SpMM, loss, Adam) + {args.precision} tensor-core GEMM operands",
            "data": "synthetic", "config": main["config"], "roofline": main["roofline"],
            "cpu_baseline": main["cpu_baseline"], "e2e": main["e2e"], "gpu_launches": main["gpu_launches"],
            "clocks": main["clocks"], "kernels": main["kernels"], "final_loss": main["final_loss"],
            "epoch_ms": main["epoch_ms"],
            "setup_s": main["setup_s"], "secondary": secondary or None,
            # SURVEY d.4: the nominal figures beside the measured ones, and the L2 size read at run time
            "device": {"l2_bytes": l2_bytes, "nominal": {"hbm_TBps": 8.0, "nvlink_GBps_per_direction": 900,
                                                         "tf32_dense_PFLOPs": 1.1, "bf16_dense_PFLOPs": 2.25}},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="reddit", choices=["cora", "pubmed", "arxiv", "reddit", "products", "nell"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--partition", default="1d", choices=["1d", "greedy", "hierarchical"],
                    help="N > 1: contiguous 1D (north star) or Alg. 4 Phase III / II-III + relabelling")
    ap.add_argument("--comm", default="p2p", choices=["nccl", "p2p"],
                    help="N > 1: NVLink peer-memory halo pulls with the gradient sum fused into the optimizer "
                         "(default; SURVEY §8(f) NEXT-1), or NCCL grouped send/recv + all-reduce")
    ap.add_argument("--aggregator", default="gcn", choices=["gcn", "sum", "mean", "max"],
                    help="aggregation scheme (SURVEY §8(f) NEXT-4; the north star's workloads are gcn)")
    ap.add_argument("--precision", default="tf32", choices=["tf32", "bf16"],
                    help="GEMM operands: TF32 (FP32 storage) or BF16 (GEMM-only tensors stored as bfloat16); "
                         "aggregation, loss and Adam are FP32 either way")
    ap.add_argument("--share-device", action="store_true",
                    help="testing only: run every rank on cuda:0 (gloo plumbing, --comm p2p) to exercise the "
                         "N > 1 path on a one-GPU box; the timings are not meaningful")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-probe", action="store_true", help="skip the gather-bandwidth probe")
    ap.add_argument("--graph", action="store_true",
                    help="time CUDA-graph replays of a captured epoch (1 GPU; launch-bound configs)")
    ap.add_argument("--secondary", default="reddit:bf16,products,products:bf16",
                    help="comma-separated extra workloads timed in the same run (device time + roofline), each "
                         "'config' or 'config:precision', or none")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
