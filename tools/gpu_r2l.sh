#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_aggregators.py tests/test_gpu_fullsize_train.py -m gpu -q -s --timeout 800 -p no:cacheprovider -k "teacher_forced_against or (reddit and (gradients or teacher))" > gpurun_out/r2l_tests.log 2>&1; echo "gpu tests rc=$?"
grep -E "passed|failed|FAILED|Error|worst|bound = |entries over" gpurun_out/r2l_tests.log | head -40
