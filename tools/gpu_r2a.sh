#!/bin/bash
# round 2: GPU suite without products-scale tests (products goldens pending), then a default bench
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
nproc > gpurun_out/r2a_nproc.txt; free -g >> gpurun_out/r2a_nproc.txt
timeout 1800 python -m pytest tests -m gpu -q -s --timeout 900 -p no:cacheprovider -k "not products" ${PYTEST_ARGS} > gpurun_out/r2a_tests.log 2>&1; echo "gpu tests rc=$?"
grep -E "passed|failed|FAILED|Error|max \|err\||epoch [0-9]+: gpu|teacher|hub degrees" gpurun_out/r2a_tests.log | head -80
timeout 600 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/r2a_bench.json
