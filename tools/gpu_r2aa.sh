#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none -k regex:k_spmm -s 6 -c 3 -o gpurun_out/r2aa_reddit python tools/profile_step.py --config reddit --epochs 2 > /dev/null 2>&1; echo "ncu rc=$?"
/usr/local/cuda/bin/ncu -i gpurun_out/r2aa_reddit.ncu-rep --page raw --csv > gpurun_out/r2aa_reddit_raw.csv 2>/dev/null
rm -f gpurun_out/r2aa_reddit.ncu-rep
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/r2aa_reddit_raw.csv")))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    print(d.get("Kernel Name", "")[:40], d.get("gpu__time_duration.sum"))
    st = {h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): float(v)
          for h, v in d.items() if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio") and v}
    tot = sum(st.values())
    for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]:
        print(f"   {k:28s} {v:6.2f} cycles/issue ({100 * v / tot:4.1f} %)")
PY
