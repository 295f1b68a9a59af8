#!/bin/bash
# round 2: aggregator teacher-forced exact bars, P2P mode-mismatch, NCCL (skips on 1 GPU); bench re-baseline
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_aggregators.py tests/test_gpu_p2p.py tests/test_gpu_nccl.py tests/test_gpu_kernels.py -m gpu -q -s --timeout 600 -p no:cacheprovider -k "teacher or mismatch or nccl or feature_switch or sparse_feature" > gpurun_out/r2c_tests.log 2>&1; echo "gpu tests rc=$?"
grep -E "passed|failed|FAILED|Error|worst|skipped" gpurun_out/r2c_tests.log | head -30
B="python bench.py --steps 20 --warmup 5 --secondary none --no-cpu-baseline --no-e2e"
for cfg in reddit products; do
  timeout 600 $B --config $cfg > gpurun_out/r2c_$cfg.json 2>gpurun_out/r2c_err.txt
  python - "$cfg" <<'PY'
import json,sys
d=json.loads(open(f"gpurun_out/r2c_{sys.argv[1]}.json").read().strip().splitlines()[-1])
k=d["kernels"]
print(sys.argv[1], round(d["value"],3), {n: round(v["ms_per_epoch"],3) for n,v in k.items()}, "frac", round(d["roofline"]["frac"],3), round(d["roofline"]["peak"]), d["roofline"].get("measured_probe_GBps"))
PY
done
