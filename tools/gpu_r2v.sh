#!/bin/bash
# round 2: 256-bit gathers — parity with the knob on, and A/B
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
MPH_SPMM_V8=1 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -m gpu -q -s --timeout 800 -p no:cacheprovider -k "spmm or hub" > gpurun_out/r2v_tests.log 2>&1; echo "gpu tests rc=$?"
grep -E "passed|failed|FAILED|Error|max \|err" gpurun_out/r2v_tests.log | head -10
timeout 600 python tools/spmm_bench.py reddit 48:48,64:128,128:128 MPH_SPMM_V8=0,1,2,3 2>&1 | tee gpurun_out/r2v_spmm_reddit.txt
timeout 600 python tools/spmm_bench.py products 48:48,104:104,128:256,256:256 MPH_SPMM_V8=0,1,2,3 2>&1 | tee gpurun_out/r2v_spmm_products.txt
