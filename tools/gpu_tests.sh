#!/bin/bash
# GPU parity suite + smoke (logs under gpurun_out/).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/t_gpu.log 2>&1; echo "gpu tests rc=$?"
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/t_gpu.log | head -30
cat gpurun_out/smoke.log | tail -3
