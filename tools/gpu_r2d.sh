#!/bin/bash
# round 2: L1-hint SpMM tests + A/B, aggregator teacher-forced bars, reddit full-size gradients (new bounds)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_aggregators.py tests/test_gpu_fullsize_train.py -m gpu -q -s --timeout 900 -p no:cacheprovider -k "hints or spmm_widths or teacher or (reddit and (gradients or teacher))" > gpurun_out/r2d_tests.log 2>&1; echo "gpu tests rc=$?"
grep -E "passed|failed|FAILED|Error|worst|max \|err\|" gpurun_out/r2d_tests.log | head -40
B="python bench.py --steps 20 --warmup 5 --secondary none --no-cpu-baseline --no-e2e --no-probe"
for cfg in reddit products; do for hot in 0 512 768 1024; do
  MPH_SPMM_HOT=$hot timeout 600 $B --config $cfg > gpurun_out/r2d_${cfg}_$hot.json 2>>gpurun_out/r2d_err.txt
  python - "$cfg" "$hot" <<'PY'
import json,sys
d=json.loads(open(f"gpurun_out/r2d_{sys.argv[1]}_{sys.argv[2]}.json").read().strip().splitlines()[-1])
k=d["kernels"]
print(sys.argv[1], "hot", sys.argv[2], round(d["value"],3), "spmm", round(k["spmm"]["ms_per_epoch"],3), "setup", d["setup_s"])
PY
done; done
tail -3 gpurun_out/r2d_err.txt
