#!/bin/bash
# round 2: full-size gradient parity against the TF32-operand oracle + teacher-forced aggregator bars
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fullsize_train.py tests/test_gpu_aggregators.py -m gpu -q -s --timeout 1200 -p no:cacheprovider -k "gradients or teacher or trajectory" > gpurun_out/r2k_tests.log 2>&1; echo "gpu tests rc=$?"
grep -E "passed|failed|FAILED|Error|tf32 oracle|worst|epoch 10" gpurun_out/r2k_tests.log | head -80
