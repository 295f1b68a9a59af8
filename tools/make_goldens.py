"""Write the full-size parity goldens (tests/golden/fullsize_<config>.npz) from the FP64 oracle.

Imports only `oracle/` and `synth/` (task ③: a stored expected value is written by a committed
script that calls only the oracle).  Nothing here touches the CUDA path.

Per config (BASELINE.json's Reddit- and ogbn-products-shaped workloads):

* ``losses`` — loss_1..loss_E of the free-running FP64 trajectory (Listing 1: forward,
  softmax-CE, backward, Adam(0.01, 0.9, 0.999), Xavier seed 42; SURVEY c.5 / Q24).
* ``g1_*`` — the epoch-1 gradients dW_l, db_l at θ_0 and their element-wise magnitude bounds
  ``bW_l = |H_{l-1}|ᵀ·(Â·M_l)`` and ``bb_l = Σ_u M_l[u]`` (the GEMM bound of SURVEY c.5,
  ``|C − C*| ≤ 2e-3·(|A|·|B|)``, composed through the aggregation: Â ≥ 0 and Âᵀ = Â make
  ``|H|ᵀ·|Â·dZ| ≤ |H|ᵀ·Â·|dZ| = (Â·|H|)ᵀ·|dZ|``, so one bound serves the transform-first product
  ``Hᵀ·(Â·dZ)`` and the aggregate-first ``(Â·H)ᵀ·dZ``).  M_l = |dZ_l| on the output layer; on a
  ReLU layer (reading Q8, ReLU'(0) := 0) the mask is a discontinuity: where the pre-activation
  lies within the forward GEMM tolerance of zero, ``|Z_l| ≤ 2e-3·Â·(|H_{l-1}|·|W_l|)``, either
  side of the mask is a correct rounding of the same product, so there the bound takes the
  unmasked gradient: ``M_l = |dZ_l| + [|Z_l| ≤ 2e-3·Â·(|H_{l-1}|·|W_l|)]·|dH_l|``.
* ``tf<t>_*`` — teacher-forced epochs: θ_{t-1} of the oracle's trajectory rounded to FP32 (what
  the GPU can hold), and the oracle's loss_t and gradients at exactly that FP32 θ, with bounds.
  These keep the check meaningful after the synthetic task's loss collapses.
* ``input_sha256`` — a digest of the generated (src, dst, X, y), so a test can tell that it
  regenerated the same inputs.

Usage: python tools/make_goldens.py reddit products [--epochs 10] [--tf 5,10]
"""
from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from synth.generate import make_workload  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")


def input_digest(w) -> str:
    h = hashlib.sha256()
    for k in ("src", "dst", "X", "y"):
        a = np.ascontiguousarray(w[k])
        h.update(k.encode())
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(memoryview(a).cast("B"))
    return h.hexdigest()


def grads_with_bounds(g, X, Ws, bs, labels):
    """loss, dWs, dbs at (Ws, bs) and the element-wise magnitude bounds (module docstring).  The
    bounds are magnitudes scaled by 2e-3 in the test, so they are formed in FP32 (relative error
    ~1e-7), layer by layer from the top, releasing the oracle's activations as they are used
    (products-sized caches are ~45 GB in FP64)."""
    import scipy.sparse as sp
    Z, cache = oracle.forward(g, X, Ws, bs)
    loss, dZ = oracle.softmax_ce(Z, labels)
    dWs, dbs = oracle.backward(g, cache, Ws, dZ)
    del Z, dZ
    A32 = sp.csr_matrix((oracle.a_hat_values(g).astype(np.float32), g.col_idx, g.row_ptr),
                        shape=(g.num_nodes, g.num_nodes))
    L = len(Ws)
    bWs, bbs = [None] * L, [None] * L
    f32 = lambda a: np.abs(np.asarray(a.toarray() if sp.issparse(a) else a)).astype(np.float32)  # noqa: E731
    for l in range(L - 1, -1, -1):
        M = f32(cache["dZ"][l])
        Hp = f32(cache["H"][l])
        if l < L - 1:   # a ReLU layer: the mask is undecided within the forward tolerance
            bz = oracle.csr_matmul(A32, Hp @ f32(Ws[l]))
            amb = np.abs(cache["Z"][l]) <= 2e-3 * bz
            del bz
            M += amb * f32(cache["dH"][l])
            del amb
        bWs[l] = (Hp.T @ oracle.csr_matmul(A32, M)).astype(np.float64)
        bbs[l] = M.sum(axis=0, dtype=np.float64)
        del M, Hp
        cache["dZ"][l] = cache["Z"][l] = cache["dH"][l] = None
        if l + 1 < len(cache["H"]):
            cache["H"][l + 1] = None
    return loss, dWs, dbs, bWs, bbs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--epochs", type=int, default=10)
    ap.add_argument("--tf", default="5,10", help="teacher-forced epochs t (θ_{t-1} from the trajectory)")
    args = ap.parse_args()
    tf_epochs = [int(x) for x in args.tf.split(",") if x]
    for name in args.configs:
        t0 = time.time()
        w = make_workload(name)
        cfg = w["cfg"]
        digest = input_digest(w)
        g = oracle.graph_build(w["src"], w["dst"], cfg.num_nodes)
        X, y, dims = w["X"], w["y"], cfg.dims
        L = len(dims) - 1
        print(f"[{name}] inputs + CSR {time.time() - t0:.1f} s", flush=True)
        out = {"input_sha256": np.array(digest), "dims": np.array(dims, np.int64), "seed": np.array(42),
               "adam": np.array([0.01, 0.9, 0.999, 1e-8])}

        # epoch-1 gradients and bounds at θ_0
        Ws, bs = oracle.xavier_init(dims, 42)
        loss1, dWs, dbs, bWs, bbs = grads_with_bounds(g, X, Ws, bs, y)
        for l in range(L):
            out[f"g1_dW{l + 1}"], out[f"g1_db{l + 1}"] = dWs[l], dbs[l]
            out[f"g1_bW{l + 1}"], out[f"g1_bb{l + 1}"] = bWs[l], bbs[l]
        print(f"[{name}] epoch-1 gradients {time.time() - t0:.1f} s (loss1 {loss1:.9f})", flush=True)

        # free-running trajectory, keeping θ_{t-1} for the teacher-forced epochs
        params = [np.asarray(a, np.float64).copy() for a in Ws] + [np.asarray(b, np.float64).copy() for b in bs]
        m = [np.zeros_like(p) for p in params]
        v = [np.zeros_like(p) for p in params]
        losses, snaps = [], {}
        for t in range(1, args.epochs + 1):
            if t in tf_epochs:
                snaps[t] = [p.astype(np.float32) for p in params]
            Z, cache = oracle.forward(g, X, params[:L], params[L:], epoch=t)
            loss, dZ = oracle.softmax_ce(Z, y)
            losses.append(loss)
            gW, gb = oracle.backward(g, cache, params[:L], dZ)
            oracle.adam_step(params, gW + gb, m, v, t)
            del Z, cache, dZ
            print(f"[{name}] epoch {t} loss {loss:.9f}  ({time.time() - t0:.1f} s)", flush=True)
        out["losses"] = np.array(losses)
        assert abs(losses[0] - loss1) <= 1e-12 * max(1.0, abs(loss1))

        # teacher-forced epochs at the FP32-rounded θ_{t-1}
        for t, th in snaps.items():
            Wt = [a.astype(np.float64) for a in th[:L]]
            bt = [b.astype(np.float64) for b in th[L:]]
            lt, dW, db, bW, bb = grads_with_bounds(g, X, Wt, bt, y)
            out[f"tf{t}_loss"] = np.array(lt)
            for l in range(L):
                out[f"tf{t}_W{l + 1}"], out[f"tf{t}_b{l + 1}"] = th[l], th[L + l]
                out[f"tf{t}_dW{l + 1}"], out[f"tf{t}_db{l + 1}"] = dW[l], db[l]
                out[f"tf{t}_bW{l + 1}"], out[f"tf{t}_bb{l + 1}"] = bW[l], bb[l]
            print(f"[{name}] teacher-forced epoch {t}: loss {lt:.9f}", flush=True)
        out["tf_epochs"] = np.array(sorted(snaps), np.int64)
        path = os.path.join(GOLDEN, f"fullsize_{name}.npz")
        np.savez_compressed(path, **out)
        print(f"[{name}] wrote {path} ({os.path.getsize(path) / 1e6:.2f} MB) in {time.time() - t0:.1f} s", flush=True)


if __name__ == "__main__":
    main()
