"""Predicted ms/epoch at P = 1/2/4/8 from the 1-GPU measurement and the partition statistics —
the paper's distributed cost model (T_epoch = T_comp + T_halo + T_grad, halo overlapped
with the local-edge aggregation) instantiated with B200 numbers.  A prediction for the
driver's scaling runs, not a measurement (this run has one GPU).

    python tools/scaling_model.py --bench profiles/r01_v9_bench_default.json \
        --partition profiles/r01_partition_compare.json --out profiles/r01_scaling_prediction.json

Per configuration and P (contiguous 1D partition, the bench default):
  * aggregation: T_spmm(1) · max_r Σd̃_r / Σd̃ (work ∝ edges of the busiest rank);
    the local-edge part (1 − cut fraction) overlaps the halo pull;
  * dense / elementwise kernels: T(1) · max_r n_r / N;
  * halo: per exchange max_r ghost_r · 4·w bytes at 770 GB/s (measured peer copy), exchanges of
    the epoch = the transform-first aggregation calls (an aggregate-first layer 1 exchanges its
    constant input once, at setup); exposed part = max(0, T_halo − T_local_part);
  * gradient sum: every rank stores |θ| floats into every other rank's slab (P2P), at 770 GB/s.
"""
from __future__ import annotations

import argparse
import json

NVLINK_GBPS = 770.0  # measured peer copy per direction on this pool (B200_PROFILING.md); 900 nominal
WIDTHS = {"reddit": ([128, 48], [0, 0]), "products": ([256, 256, 48], [1, 0, 0])}  # pout per layer, order
PARAMS = {"reddit": 602 * 128 + 128 + 128 * 48 + 48, "products": 104 * 256 + 256 + 256 * 256 + 256 + 256 * 48 + 48}


def predict(cfg, bench_line, part_case):
    k = bench_line["kernels"]
    t_spmm = k["spmm"]["ms_per_epoch"]
    t1 = bench_line["value"]
    # everything but the aggregation, as wall time (weight-gradient GEMMs may overlap on a side stream)
    t_dense = max(0.0, t1 - t_spmm)
    t_other = 0.0
    pout, order = WIDTHS[cfg]
    xchg_widths = [w for w, o in zip(pout, order) if o == 0] * 2          # forward + backward per TF layer
    rows = []
    for world in ("1", "2", "4", "8"):
        if world == "1":
            rows.append({"P": 1, "ms_epoch": t1, "spmm": t_spmm, "dense": t_dense, "halo_exposed": 0.0, "grad": 0.0})
            continue
        st = part_case["by_world"][world]["1d"]
        per = st["per_rank"]                      # [owned, sum deg~, ghosts, cut entries]
        n_tot = sum(r[0] for r in per)
        d_tot = sum(r[1] for r in per)
        spmm = t_spmm * max(r[1] for r in per) / d_tot
        dense = (t_dense + t_other) * max(r[0] for r in per) / n_tot
        cut = st["cut_fraction"]
        ghost_max = max(r[2] for r in per)
        halo = sum(ghost_max * 4.0 * w / (NVLINK_GBPS * 1e6) for w in xchg_widths)
        local = spmm * (1.0 - cut) * len(xchg_widths) / max(1, len(xchg_widths) + order.count(1))
        exposed = max(0.0, halo - local)
        grad = PARAMS[cfg] * 4.0 * (int(world) - 1) / (NVLINK_GBPS * 1e6)
        rows.append({"P": int(world), "ms_epoch": spmm + dense + exposed + grad, "spmm": spmm, "dense": dense,
                     "halo_total": halo, "halo_exposed": exposed, "grad": grad, "ghost_rows_max": ghost_max,
                     "cut_fraction": cut})
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bench", required=True)
    ap.add_argument("--partition", default="profiles/r01_partition_compare.json")
    ap.add_argument("--out", default="profiles/r01_scaling_prediction.json")
    a = ap.parse_args()
    b = json.load(open(a.bench))
    parts = {c["graph"]: c for c in json.load(open(a.partition))["cases"]}
    lines = {"reddit": b}
    lines.update({name: r for name, r in (b.get("secondary") or {}).items() if ":" not in name})
    out = {"what": "predicted ms/epoch (cost model P:545-569 with B200 rates); not a measurement",
           "bench": a.bench, "nvlink_GBps": NVLINK_GBPS, "configs": {}}
    for cfg in ("reddit", "products"):
        if cfg in lines and cfg in parts:
            out["configs"][cfg] = predict(cfg, lines[cfg], parts[cfg])
            for r in out["configs"][cfg]:
                print(cfg, r["P"], round(r["ms_epoch"], 3), "ms  speedup", round(out["configs"][cfg][0]["ms_epoch"] /
                                                                            r["ms_epoch"], 2),
                      " halo exposed", round(r.get("halo_exposed", 0.0), 3))
    with open(a.out, "w") as fh:
        json.dump(out, fh, indent=1)
        fh.write("\n")


if __name__ == "__main__":
    main()
