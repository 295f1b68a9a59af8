#!/bin/bash
# Quick A/B on the GPU: selected parity tests + device-timed bench of several configs (no e2e, no CPU leg).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-ab}
TESTS=${2:-"spmm or softmax or localized or fullsize or trajectory"}
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider -k "$TESTS" > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${TAG}_tests.log
for c in ${CONFIGS:-reddit products arxiv}; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-probe --secondary none \
    > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err; echo "bench $c rc=$?"
  python - $TAG $c <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/{sys.argv[1]}_bench_{sys.argv[2]}.json"))
print(sys.argv[2], round(d["value"], 3), "ms/epoch", {k: round(v["ms_per_epoch"], 3) for k, v in d["kernels"].items()})
PY
done
