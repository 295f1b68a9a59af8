#!/bin/bash
# round 2: new parity tests (products full size, L1 hints), then bench A/B of the SpMM knobs
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fullsize_train.py tests/test_gpu_fullsize.py tests/test_gpu_kernels.py -m gpu -q -s --timeout 900 -p no:cacheprovider -k "products or hints or hub" > gpurun_out/r2b_tests.log 2>&1; echo "gpu tests rc=$?"
grep -E "passed|failed|FAILED|Error|max \|err\||epoch [0-9]+: gpu|teacher" gpurun_out/r2b_tests.log | head -60
B="python bench.py --steps 20 --warmup 5 --secondary none --no-cpu-baseline --no-e2e"
for hot in 0 512 768 1024; do
  MPH_SPMM_HOT=$hot timeout 600 $B --config reddit > gpurun_out/r2b_reddit_hot$hot.json 2>gpurun_out/r2b_err.txt
  python - "$hot" <<'PY'
import json,sys
d=json.loads(open(f"gpurun_out/r2b_reddit_hot{sys.argv[1]}.json").read().strip().splitlines()[-1])
print("reddit hot", sys.argv[1], round(d["value"],3), "spmm", round(d["kernels"]["spmm"]["ms_per_epoch"],3), "frac", round(d["roofline"]["frac"],3), d["roofline"]["peak"])
PY
done
for hot in 0 384 768; do for rows in 0 1; do
  MPH_SPMM_HOT=$hot MPH_SPMM_ROWS=$rows timeout 600 $B --config products > gpurun_out/r2b_products_hot${hot}_rows$rows.json 2>>gpurun_out/r2b_err.txt
  python - "$hot" "$rows" <<'PY'
import json,sys
d=json.loads(open(f"gpurun_out/r2b_products_hot{sys.argv[1]}_rows{sys.argv[2]}.json").read().strip().splitlines()[-1])
print("products hot", sys.argv[1], "rows", sys.argv[2], round(d["value"],3), "spmm", round(d["kernels"]["spmm"]["ms_per_epoch"],3))
PY
done; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2b_ref.json 2>>gpurun_out/r2b_err.txt; tail -c 600 gpurun_out/r2b_ref.json
tail -5 gpurun_out/r2b_err.txt
