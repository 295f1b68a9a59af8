"""Per-launch table (time, DRAM read/write, GB/s) from an `ncu --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv` log (lines before the CSV header are skipped)."""
import csv
import io
import sys

text = open(sys.argv[1]).read()
text = text[text.index('"ID"'):]
by = {}
for r in csv.DictReader(io.StringIO(text)):
    k = (int(r["ID"]), r["Kernel Name"].split("(")[0][-40:], r["Block Size"], r["Grid Size"])
    by.setdefault(k, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
for (i, n, b, g), m in sorted(by.items()):
    t = m["gpu__time_duration.sum"]
    rd, wr = m.get("dram__bytes_read.sum", 0.0), m.get("dram__bytes_write.sum", 0.0)
    print(f"{i:3d} {n:40s} {b:12s} {g:12s} {t / 1e3:9.1f} us  rd {rd / 1e9:6.2f} GB  wr {wr / 1e9:6.2f} GB  "
          f"{(rd + wr) / t:7.0f} GB/s")
