"""Write the full-size parity goldens (tests/golden/fullsize_<config>.npz) from the FP64 oracle.

Imports only `oracle/` and `synth/` (task ③: a stored expected value is written by a committed
script that calls only the oracle).  Nothing here touches the CUDA path.

Per config (BASELINE.json's Reddit- and ogbn-products-shaped workloads):

* ``losses`` — loss_1..loss_E of the free-running FP64 trajectory (Listing 1: forward,
  softmax-CE, backward, Adam(0.01, 0.9, 0.999), Xavier seed 42; SURVEY c.5 / Q24).
* ``g1_*`` — the epoch-1 gradients dW_l, db_l of the exact oracle at θ_0 (compared normwise,
  reading R1).
* ``g1t_*`` — the same gradients from the oracle with the kernel's operand rounding
  (``operand_rounding="tf32"``, reading R2: both operands of every dense product rounded to TF32
  as the GPU stores them, in the GPU's layer orders, reading Q7), with the element-wise bounds of
  ``oracle.tf32_gradient_bounds`` (oracle/bounds.py): the GEMM bound of each weight-gradient
  product, ``2e-3·|A_l|ᵀ·|B_l|`` for ``dW_l = A_lᵀ·B_l`` (SURVEY c.5 "gradients can be compared after
  step 1 with the GEMM bound", the north star's 2e-3 applied to one product), plus the ReLU
  decisions FP32 accumulation can flip.  With the operand rounding on both sides what remains
  between GPU and oracle is FP32 accumulation order; against the EXACT oracle the TF32 error of
  every upstream product feeds each dW through cancelling sums, which no single-product bound
  covers (measured: 5-40x over it on products' layer 2), hence the two references.
* ``tf<t>_*`` / ``tf<t>t_*`` — teacher-forced epochs: θ_{t-1} of the oracle's trajectory rounded
  to FP32 (what the GPU can hold), and both oracles' loss_t and gradients at exactly that FP32 θ
  (bounds as above).  These keep the check meaningful after the synthetic task's loss collapses.
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


def layer_orders(dims, dense_features=True):
    """The GPU's layer orders (reading Q7): layer 1 aggregate-first iff its features are
    dense and F_1 > F_0; every other layer transform-first."""
    return tuple("AF" if (l == 0 and dense_features and dims[1] > dims[0]) else "TF" for l in range(len(dims) - 1))


def exact_grads(g, X, Ws, bs, labels):
    """loss, dWs, dbs of the exact FP64 oracle at (Ws, bs)."""
    Z, cache = oracle.forward(g, X, Ws, bs)
    loss, dZ = oracle.softmax_ce(Z, labels)
    dWs, dbs = oracle.backward(g, cache, Ws, dZ)
    return loss, dWs, dbs


def tf32_grads_with_bounds(g, X, Ws, bs, labels, orders):
    """loss, dWs, dbs of the TF32-operand oracle and oracle.tf32_gradient_bounds, formed in FP32
    (a tolerance), releasing the activations as they are used (products-sized FP64 caches are
    ~45 GB)."""
    Z, cache = oracle.forward(g, X, Ws, bs, operand_rounding="tf32", orders=orders)
    loss, dZ = oracle.softmax_ce(Z, labels)
    dWs, dbs = oracle.backward(g, cache, Ws, dZ)
    del Z, dZ
    cache["Z"][-1] = None   # the output layer's Z is not needed by the bound (no ReLU)
    for key in ("H", "Z", "Y", "dZ", "dH"):   # a tolerance needs no FP64: halve the ~45 GB cache
        for i, a in enumerate(cache[key]):
            if isinstance(a, np.ndarray) and a.dtype == np.float64:
                cache[key][i] = a.astype(np.float32)
                del a
    bWs, bbs = oracle.tf32_gradient_bounds(g, cache, Ws, bs, release=True, dtype=np.float32)
    return loss, dWs, dbs, bWs, bbs


def _eval_main(argv):
    """--eval <config> <theta.npz> <out.npz> <exact|tf32>: one gradient evaluation in a fresh
    process (regenerates the inputs), so the ~45 GB of FP64 activations of a products-sized
    evaluation never share a heap with the trajectory (the host has 62 GB)."""
    name, src, dst, kind = argv
    w = make_workload(name)
    g = oracle.graph_build(w["src"], w["dst"], w["cfg"].num_nodes)
    th = dict(np.load(src))
    L = len(w["cfg"].dims) - 1
    Ws = [th[f"W{l}"] for l in range(L)]
    bs = [th[f"b{l}"] for l in range(L)]
    if kind == "exact":
        loss, dW, db = exact_grads(g, w["X"], Ws, bs, w["y"])
        bW = bb = [np.zeros(0)] * L
    else:
        loss, dW, db, bW, bb = tf32_grads_with_bounds(g, w["X"], Ws, bs, w["y"], layer_orders(w["cfg"].dims))
    out = {"loss": np.array(loss)}
    for l in range(L):
        out[f"dW{l}"], out[f"db{l}"], out[f"bW{l}"], out[f"bb{l}"] = dW[l], db[l], bW[l], bb[l]
    np.savez(dst, **out)


def _in_child(name, kind, Ws, bs):
    import subprocess
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        src, dst = os.path.join(d, "theta.npz"), os.path.join(d, "out.npz")
        np.savez(src, **{f"W{l}": np.asarray(W) for l, W in enumerate(Ws)},
                 **{f"b{l}": np.asarray(b) for l, b in enumerate(bs)})
        subprocess.run([sys.executable, os.path.abspath(__file__), "--eval", name, src, dst, kind], check=True)
        r = dict(np.load(dst))
    L = len(Ws)
    dW = [r[f"dW{l}"] for l in range(L)]
    db = [r[f"db{l}"] for l in range(L)]
    if kind == "exact":
        return float(r["loss"]), dW, db
    return float(r["loss"]), dW, db, [r[f"bW{l}"] for l in range(L)], [r[f"bb{l}"] for l in range(L)]


def _traj_main(argv):
    """--traj <config> <epochs> <t1,t2,..> <out.npz>: the free-running FP64 trajectory (Listing 1
    P:159-173) in a fresh process; writes the losses and θ_{t-1} (FP32) for each teacher-forced t."""
    name, epochs, tfs, dst = argv[0], int(argv[1]), [int(x) for x in argv[2].split(",") if x], argv[3]
    w = make_workload(name)
    g = oracle.graph_build(w["src"], w["dst"], w["cfg"].num_nodes)
    X, y, dims = w["X"], w["y"], w["cfg"].dims
    L = len(dims) - 1
    Ws, bs = oracle.xavier_init(dims, 42)
    params = [np.asarray(a, np.float64).copy() for a in Ws] + [np.asarray(b, np.float64).copy() for b in bs]
    m = [np.zeros_like(p) for p in params]
    v = [np.zeros_like(p) for p in params]
    out = {}
    losses = []
    for t in range(1, epochs + 1):
        if t in tfs:
            for i, p in enumerate(params):
                out[f"s{t}_{i}"] = p.astype(np.float32)
        Z, cache = oracle.forward(g, X, params[:L], params[L:], epoch=t)
        loss, dZ = oracle.softmax_ce(Z, y)
        losses.append(loss)
        gW, gb = oracle.backward(g, cache, params[:L], dZ)
        oracle.adam_step(params, gW + gb, m, v, t)
        del Z, cache, dZ
        print(f"[{name}] epoch {t} loss {loss:.9f}", flush=True)
    out["losses"] = np.array(losses)
    np.savez(dst, **out)


def _traj_in_child(name, epochs, tfs, L):
    import subprocess
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        dst = os.path.join(d, "traj.npz")
        subprocess.run([sys.executable, os.path.abspath(__file__), "--traj", name, str(epochs),
                        ",".join(str(t) for t in tfs), dst], check=True)
        r = dict(np.load(dst))
    snaps = {t: [r[f"s{t}_{i}"] for i in range(2 * L)] for t in tfs if f"s{t}_0" in r}
    return [float(x) for x in r["losses"]], snaps


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
        dims = cfg.dims
        L = len(dims) - 1
        del w   # every evaluation below runs in a fresh process (_in_child / _traj_in_child)
        out = {"input_sha256": np.array(digest), "dims": np.array(dims, np.int64), "seed": np.array(42),
               "adam": np.array([0.01, 0.9, 0.999, 1e-8])}

        orders = layer_orders(dims)
        out["orders"] = np.array(orders)

        # epoch-1 gradients at θ_0: exact, and TF32-operand with bounds
        Ws, bs = oracle.xavier_init(dims, 42)
        loss1, dWs, dbs = _in_child(name, "exact", Ws, bs)
        for l in range(L):
            out[f"g1_dW{l + 1}"], out[f"g1_db{l + 1}"] = dWs[l], dbs[l]
        lt1, dWs, dbs, bWs, bbs = _in_child(name, "tf32", Ws, bs)
        for l in range(L):
            out[f"g1t_dW{l + 1}"], out[f"g1t_db{l + 1}"] = dWs[l], dbs[l]
            out[f"g1t_bW{l + 1}"], out[f"g1t_bb{l + 1}"] = bWs[l], bbs[l]
        out["g1t_loss"] = np.array(lt1)
        print(f"[{name}] epoch-1 gradients {time.time() - t0:.1f} s (loss1 {loss1:.9f}, tf32 {lt1:.9f})", flush=True)

        # free-running trajectory, keeping θ_{t-1} for the teacher-forced epochs
        losses, snaps = _traj_in_child(name, args.epochs, tf_epochs, L)
        out["losses"] = np.array(losses)
        print(f"[{name}] trajectory {time.time() - t0:.1f} s: " + " ".join(f"{x:.6g}" for x in losses), flush=True)
        assert abs(losses[0] - loss1) <= 1e-12 * max(1.0, abs(loss1))

        # teacher-forced epochs at the FP32-rounded θ_{t-1}
        for t, th in snaps.items():
            Wt = [a.astype(np.float64) for a in th[:L]]
            bt = [b.astype(np.float64) for b in th[L:]]
            lt, dW, db = _in_child(name, "exact", Wt, bt)
            out[f"tf{t}_loss"] = np.array(lt)
            for l in range(L):
                out[f"tf{t}_W{l + 1}"], out[f"tf{t}_b{l + 1}"] = th[l], th[L + l]
                out[f"tf{t}_dW{l + 1}"], out[f"tf{t}_db{l + 1}"] = dW[l], db[l]
            lr, dW, db, bW, bb = _in_child(name, "tf32", Wt, bt)
            out[f"tf{t}t_loss"] = np.array(lr)
            for l in range(L):
                out[f"tf{t}t_dW{l + 1}"], out[f"tf{t}t_db{l + 1}"] = dW[l], db[l]
                out[f"tf{t}t_bW{l + 1}"], out[f"tf{t}t_bb{l + 1}"] = bW[l], bb[l]
            print(f"[{name}] teacher-forced epoch {t}: loss {lt:.9f}", flush=True)
        out["tf_epochs"] = np.array(sorted(snaps), np.int64)
        path = os.path.join(GOLDEN, f"fullsize_{name}.npz")
        np.savez_compressed(path, **out)
        print(f"[{name}] wrote {path} ({os.path.getsize(path) / 1e6:.2f} MB) in {time.time() - t0:.1f} s", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--eval":
        _eval_main(sys.argv[2:])
    elif len(sys.argv) > 1 and sys.argv[1] == "--traj":
        _traj_main(sys.argv[2:])
    else:
        main()
