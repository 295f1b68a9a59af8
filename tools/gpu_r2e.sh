#!/bin/bash
# round 2: L2-tag SpMM test + products A/B; ncu L2 peak metrics of the reddit SpMM and the probes
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -s --timeout 600 -p no:cacheprovider -k "l2_tags or spmm_widths" > gpurun_out/r2e_tests.log 2>&1; echo "gpu tests rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2e_tests.log | head -20
B="python bench.py --steps 20 --warmup 5 --secondary none --no-cpu-baseline --no-e2e --no-probe"
for mode in 0 1 2 3; do
  MPH_SPMM_L2TAG=$mode timeout 600 $B --config products > gpurun_out/r2e_products_$mode.json 2>>gpurun_out/r2e_err.txt
  python - "$mode" <<'PY'
import json,sys
d=json.loads(open(f"gpurun_out/r2e_products_{sys.argv[1]}.json").read().strip().splitlines()[-1])
k=d["kernels"]
print("products l2tag", sys.argv[1], round(d["value"],3), "spmm", round(k["spmm"]["ms_per_epoch"],3), "setup", d["setup_s"])
PY
done
# L2 peak as ncu defines it, from the reddit SpMM launches and the two probes
timeout 900 ncu --metrics gpu__time_duration.sum,lts__t_bytes.sum,lts__t_bytes.sum.per_second,lts__t_bytes.sum.peak_sustained,lts__cycles_elapsed.avg.per_second,lts__t_sectors.sum.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__t_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_spmm|k_probe" -c 24 --csv --log-file gpurun_out/r2e_ncu_l2.csv python bench.py --steps 2 --warmup 1 --secondary none --no-cpu-baseline --no-e2e > gpurun_out/r2e_ncu_bench.log 2>&1; echo "ncu rc=$?"
python tools/ncu_l2_peak.py gpurun_out/r2e_ncu_l2.csv
