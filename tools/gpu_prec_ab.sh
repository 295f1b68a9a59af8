#!/bin/bash
# TF32 vs BF16 GEMM operands, device-timed, on several configs.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for c in ${CONFIGS:-reddit products arxiv}; do
  for p in tf32 bf16; do
    timeout 900 python bench.py --config $c --precision $p --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-probe \
      --secondary none > gpurun_out/prec_${p}_$c.json 2> gpurun_out/prec_${p}_$c.err
    python - $p $c <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/prec_{sys.argv[1]}_{sys.argv[2]}.json"))
print(sys.argv[2], sys.argv[1], round(d["value"], 3), "ms/epoch", {k: round(v["ms_per_epoch"], 3) for k, v in d["kernels"].items()})
PY
  done
done
