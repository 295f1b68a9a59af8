"""Summarise ncu reports (.ncu-rep --set full) and launch lists into profiles/.

    python tools/ncu_summary.py gpurun_out/prof_spmm_reddit.ncu-rep [...] --out profiles/r01_ncu_summary.md
    python tools/ncu_summary.py --launches gpurun_out/launches_reddit.csv --out profiles/r01_launches_reddit.md
"""
import argparse
import csv
import io
import json
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 % peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
]


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def summarise(reps):
    lines = ["| report | kernel | " + " | ".join(n for _, n in METRICS) + " | DRAM bytes/launch |",
             "|---|---|" + "---|" * len(METRICS) + "---|"]
    data = []
    for rep in reps:
        hdr, units, rows = raw_rows(rep)
        ki = hdr.index("Kernel Name")
        for r in rows:
            vals = []
            rec = {"report": rep, "kernel": r[ki]}
            for m, _ in METRICS:
                if m in hdr:
                    i = hdr.index(m)
                    vals.append(f"{r[i]} {units[i]}".strip())
                    rec[m] = (r[i], units[i])
                else:
                    vals.append("n/a")
            def as_bytes(m):
                v, u = rec.get(m, ("0", "byte"))
                v = float(v.replace(",", ""))
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            db = as_bytes("dram__bytes_read.sum") + as_bytes("dram__bytes_write.sum")
            rec["dram_bytes_per_launch"] = db
            data.append(rec)
            name = r[ki].split("(")[0].replace("void ", "").replace("mph::", "")[:40]
            lines.append(f"| {rep.split('/')[-1]} | `{name}` | " + " | ".join(vals) + f" | {db:.4g} |")
    return "\n".join(lines), data


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = {}
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        n = r[ki].split("(")[0].replace("void ", "")
        c = tot.setdefault(n, [0, 0.0])
        c[0] += 1
        c[1] += float(r[vi].replace(",", ""))
    total = sum(v[1] for v in tot.values())
    lines = ["| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k[:60]}` | {v[0]} | {v[1] / 1e6:.3f} | {100 * v[1] / total:.1f} % |")
    return "\n".join(lines)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("reports", nargs="*")
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    ap.add_argument("--json")
    ap.add_argument("--title", default="")
    a = ap.parse_args()
    with open(a.out, "w") as f:
        if a.title:
            f.write(f"# {a.title}\n\n")
        if a.launches:
            f.write(launches(a.launches) + "\n")
        if a.reports:
            md, data = summarise(a.reports)
            f.write(md + "\n")
            if a.json:
                with open(a.json, "w") as g:
                    json.dump(data, g, indent=1)
    print(open(a.out).read())
