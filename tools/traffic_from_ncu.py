"""Regenerate profiles/ncu_traffic_<config>.json (the `traffic` field of bench.py's roofline) from
an `ncu --set full` summary JSON (tools/ncu_summary.py): the DRAM read+write bytes of one epoch's
k_spmm launches (the capture windows of tools/gpu_profile.sh cover exactly one epoch), divided by
the aggregation calls per epoch (bench.py's launch unit: a w = 128/256 row split into two column
slabs is one call of two kernels)."""
import json
import sys

summary = sys.argv[1]          # profiles/r01_vN_ncu_full.json
tag = summary.split("/")[-1].replace("_ncu_full.json", "")
CALLS = {"reddit": 4, "products": 5}
rows = json.load(open(summary))
for cfg, calls in CALLS.items():
    launches = [r for r in rows if r["report"].endswith(f"_spmm_{cfg}.ncu-rep") and "k_spmm" in r["kernel"]]
    total = sum(r["dram_bytes_per_launch"] for r in launches)
    out = {"spmm": {"dram_bytes_per_launch": total / calls,
                    "source": f"profiles/{tag}_ncu_full.md: DRAM read+write of the {len(launches)} k_spmm kernels of "
                              f"one {cfg} epoch ({total / 1e9:.2f} GB) / {calls} aggregation calls"}}
    with open(f"profiles/ncu_traffic_{cfg}.json", "w") as fh:
        json.dump(out, fh)
        fh.write("\n")
    print(cfg, out)
