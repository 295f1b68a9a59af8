"""B200 calibration of the efficiency ratio γ = η_sparse / η_dense and the switch threshold τ = 1 − γ
(Eq. 1; derivation P:232-246).

The paper measured γ ≈ 0.20 offline on its testbed and ships τ ≈ 0.80 as a heuristic.
Here the same offline microbenchmark runs on the layer-1 pair that the switch actually chooses
between, through the C-ABI:

  dense : T = X·W   (mph_gemm_nt, tcgen05)     + dW = Xᵀ·G (mph_gemm_tn, tcgen05)
  sparse: T = X_csr·W (mph_sparse_xw)          + dW = X_cscᵀ·G (mph_sparse_xtg)

for X of shape N×F at sparsity s, hidden width H.  Work terms follow P:236-240:
W_dense = 2·(2NFH) (forward + backward), W_sparse = 2·(2(1−s)NFH); η = W / T; γ(s) = η_sparse/η_dense.
The crossover s* is where T_sparse(s) = T_dense (linear interpolation between measured s);
τ_B200 = s*, γ_B200 = 1 − s*.  Every op is timed with CUDA events on the launching stream, after
warm-up, with a 512 MB L2 flush before each launch (inputs are cold, as in a training step).

Usage (GPU box):  python tools/calibrate_gamma.py [--out profiles/r01_gamma_calibration.json]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2512_01678_b200 as P  # noqa: E402
from paper_2512_01678_b200 import _lib as L  # noqa: E402
from synth.generate import make_features_csr, make_labels  # noqa: E402

SHAPES = [  # (name, N, F, H, densities of X = 1 - s)
    ("N131072_F512_H128", 131072, 512, 128, [0.7, 0.5, 0.4, 0.3, 0.2, 0.1, 0.05, 0.01]),
    ("N65536_F2048_H32", 65536, 2048, 32, [0.7, 0.5, 0.4, 0.3, 0.2, 0.1, 0.05, 0.01]),
    ("N65536_F1024_H64", 65536, 1024, 64, [0.5, 0.3, 0.2, 0.1, 0.05, 0.01]),
    ("nell_N65755_F61278_H32", 65755, 61278, 32, [0.0079]),
]


def _timed(fn, flush, reps):
    s = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    fn()
    torch.cuda.synchronize()
    for a, b in ev:
        flush.add_(1.0)
        a.record(s)
        fn()
        b.record(s)
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev]))


def uniform_csr(N, F, density, seed):
    """Bernoulli(density) binary mask in CSR form, built in row chunks (exact per-entry density;
    NELL's shape goes through synth.make_features_csr instead, as in the workload)."""
    rng = np.random.default_rng(seed)
    ptr = np.zeros(N + 1, dtype=np.int64)
    idx = []
    chunk = max(1, (1 << 26) // F)
    for r0 in range(0, N, chunk):
        m = rng.random((min(N, r0 + chunk) - r0, F), dtype=np.float32) < density
        ptr[r0 + 1:r0 + 1 + m.shape[0]] = np.count_nonzero(m, axis=1)
        idx.append(np.nonzero(m)[1].astype(np.int32))
    np.cumsum(ptr, out=ptr)
    idx = np.concatenate(idx)
    return ptr, idx, np.ones(idx.size, dtype=np.float32)


def measure_shape(name, N, F, H, densities, reps, flush):
    sid = torch.cuda.current_stream().cuda_stream
    y = make_labels(N, 16)
    rng = np.random.default_rng(0)
    W = torch.from_numpy(rng.standard_normal((F, H)).astype(np.float32)).cuda()
    G = torch.from_numpy(rng.standard_normal((N, H)).astype(np.float32)).cuda()
    ones = torch.ones(N, device="cuda")
    T = torch.empty((N, H), device="cuda")
    dW = torch.empty((F, H), device="cuda")
    Wt = W.t().contiguous()
    rows = []
    t_dense = None
    for d in densities:
        if F > 8192:
            ptr, idx, val = make_features_csr(N, F, y, 16, d, seed=int(d * 1e4) + F)
        else:
            ptr, idx, val = uniform_csr(N, F, d, seed=int(d * 1e4) + F)
        nnz = int(val.size)
        fs = P.Features.from_csr(ptr, idx, val, (N, F), force_mode=1)

        def sparse():
            L.mph_sparse_xw(fs.h, W.data_ptr(), H, H, ones.data_ptr(), T.data_ptr(), H, sid)
            L.mph_sparse_xtg(fs.h, G.data_ptr(), H, H, dW.data_ptr(), H, sid)

        t_sp = _timed(sparse, flush, reps)
        del fs
        if t_dense is None or len(densities) == 1:
            fd = P.Features.from_csr(ptr, idx, val, (N, F), force_mode=0)
            X = fd.dense()
            ld = X.shape[1]
            Wtp = torch.zeros((H, ld), device="cuda")
            Wtp[:, :F] = Wt
            wsb = C.c_size_t()
            L.mph_gemm_tn_workspace(F, H, N, C.byref(wsb))
            ws = torch.empty(max(1, wsb.value // 4), device="cuda")

            def dense():
                L.mph_gemm_nt(N, H, F, X.data_ptr(), ld, Wtp.data_ptr(), ld, T.data_ptr(), H, None, sid)
                L.mph_gemm_tn(F, H, N, X.data_ptr(), ld, G.data_ptr(), H, dW.data_ptr(), H, ws.data_ptr(), wsb.value,
                              sid)

            t_dense = _timed(dense, flush, reps)
            del fd, X, Wtp, ws
        s = 1.0 - nnz / (N * F)
        w_dense = 2 * 2.0 * N * F * H
        w_sparse = 2 * 2.0 * (1.0 - s) * N * F * H
        eta_d = w_dense / (t_dense * 1e-3)
        eta_s = w_sparse / (t_sp * 1e-3)
        rows.append({"s": s, "nnz": nnz, "t_dense_ms": t_dense, "t_sparse_ms": t_sp,
                     "eta_dense_tflops": eta_d / 1e12, "eta_sparse_tflops": eta_s / 1e12, "gamma": eta_s / eta_d,
                     "sparse_faster": t_sp < t_dense})
        print(f"{name} s={s:.4f} nnz={nnz} dense {t_dense:.3f} ms sparse {t_sp:.3f} ms gamma {eta_s / eta_d:.3f}",
              flush=True)
    cross = None
    rs = sorted(rows, key=lambda r: r["s"])
    for a, b in zip(rs, rs[1:]):
        da, db = a["t_sparse_ms"] - a["t_dense_ms"], b["t_sparse_ms"] - b["t_dense_ms"]
        if da >= 0 > db or da > 0 >= db:
            cross = a["s"] + (b["s"] - a["s"]) * da / (da - db)
    if cross is None and rs and all(r["sparse_faster"] for r in rs):
        cross = f"<= {rs[0]['s']:.3f}"
    return {"shape": name, "N": N, "F": F, "H": H, "rows": rows, "crossover_s": cross,
            "gamma_b200": (1.0 - cross) if isinstance(cross, float) else None}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/r01_gamma_calibration.json")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--shapes", default="all")
    a = ap.parse_args()
    flush = torch.zeros(128 << 20, device="cuda")  # 512 MB > 126 MB L2
    res = []
    for sh in SHAPES:
        if a.shapes != "all" and sh[0] not in a.shapes.split(","):
            continue
        res.append(measure_shape(*sh, a.reps, flush))
    crosses = [r["crossover_s"] for r in res if isinstance(r["crossover_s"], float)]
    out = {"what": "gamma/tau calibration of the layer-1 dense/sparse pair (Eq. 1, P:212-246)",
           "paper": {"gamma": 0.20, "tau": 0.80, "source": "P:216"},
           "device": torch.cuda.get_device_name(0), "shapes": res,
           "tau_b200_median": float(np.median(crosses)) if crosses else None}
    if crosses:
        out["gamma_b200_median"] = 1.0 - out["tau_b200_median"]
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "shapes"}))


if __name__ == "__main__":
    main()
