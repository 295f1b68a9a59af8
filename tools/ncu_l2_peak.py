"""L2 (LTS) throughput peak from an ncu metrics CSV: per kernel launch, lts__t_bytes / duration
against lts__t_bytes.sum.peak_sustained x lts__cycles_elapsed.avg.per_second (the hardware's
sustained LTS byte rate as ncu defines it).  Usage: python tools/ncu_l2_peak.py launches.csv [out.json]"""
import csv
import json
import sys
from collections import defaultdict

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "byte/second": 1.0, "Kbyte/second": 1e3, "Mbyte/second": 1e6, "Gbyte/second": 1e9, "Tbyte/second": 1e12,
         "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0, "s": 1.0,
         "cycle/second": 1.0, "cycle/nsecond": 1e9, "cycle/usecond": 1e6, "Ghz": 1e9, "Mhz": 1e6, "hz": 1.0,
         "byte/cycle": 1.0, "%": 1.0, "": 1.0}


def load(path):
    rows = defaultdict(dict)
    names = {}
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        key = r["ID"]
        names[key] = r["Kernel Name"]
        try:
            v = float(r["Metric Value"].replace(",", ""))
        except ValueError:
            continue
        rows[key][r["Metric Name"]] = v * SCALE.get(r["Metric Unit"], 1.0)
    return rows, names


def main():
    rows, names = load(sys.argv[1])
    out = []
    for k in sorted(rows, key=int):
        m = rows[k]
        t = m.get("gpu__time_duration.sum")
        b = m.get("lts__t_bytes.sum")
        ps, clk = m.get("lts__t_bytes.sum.peak_sustained"), m.get("lts__cycles_elapsed.avg.per_second")
        peak = ps * clk if ps and clk else None
        rate = b / t if b and t else None
        rec = {"id": int(k), "kernel": names[k][:60], "ms": t * 1e3 if t else None,
               "lts_GBps": rate / 1e9 if rate else None, "lts_peak_GBps": peak / 1e9 if peak else None,
               "lts_frac": rate / peak if rate and peak else None,
               "lts_throughput_pct": m.get("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
               "l1_bytes": m.get("l1tex__t_bytes.sum"), "lts_bytes": b,
               "dram_bytes": (m.get("dram__bytes_read.sum") or 0) + (m.get("dram__bytes_write.sum") or 0)}
        out.append(rec)
        print(json.dumps(rec))
    if len(sys.argv) > 2:
        with open(sys.argv[2], "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
