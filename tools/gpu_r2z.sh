#!/bin/bash
# round 2: sign-byte ReLU masks — parity, bitwise A/B against the value-mask build, timing
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_e2e.py tests/test_gpu_bf16.py tests/test_gpu_p2p.py tests/test_gpu_aggregators.py -m gpu -q -p no:cacheprovider --timeout 900 -k "not fullsize" > gpurun_out/r2z_tests.log 2>&1; echo "gpu tests rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2z_tests.log | head -10
bash tools/gpu_ab_build.sh "-DMPH_NO_SIGNBYTES" "python tools/loss_digest.py arxiv 6; python tools/loss_digest.py products 3; python tools/env_sweep.py products MPH_X=0 2>&1 | tail -2; python tools/env_sweep.py arxiv MPH_X=0 2>&1 | tail -2; python tools/env_sweep.py reddit MPH_X=0 2>&1 | tail -2"
