#!/bin/bash
# round 2: the other BASELINE configs (device ms/epoch, eager and CUDA-graph replay, TF32 / BF16)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for c in cora pubmed arxiv nell; do
  for extra in "" "--graph" "--precision bf16"; do
    if [ "$c" = "nell" ] && [ "$extra" = "--precision bf16" ]; then continue; fi
    timeout 600 python bench.py --config $c --steps 30 --warmup 5 --secondary none --no-cpu-baseline --no-e2e --no-probe $extra > gpurun_out/r2x_${c}${extra// /}.json 2>/dev/null
    python - "$c" "$extra" <<'PY'
import json, sys
c, extra = sys.argv[1], sys.argv[2]
d = json.loads(open(f"gpurun_out/r2x_{c}{extra.replace(' ', '')}.json").read().strip().splitlines()[-1])
k = {n: round(v["ms_per_epoch"], 3) for n, v in d["kernels"].items()}
print(c, extra or "eager", round(d["value"], 3), k, d["config"].get("layer_order"))
PY
  done
done
