#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
MPH_SPMM_CTAITEMS=8 timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -s --timeout 800 -p no:cacheprovider -k "spmm" > gpurun_out/r2p_tests.log 2>&1; echo "gpu tests rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2p_tests.log | head -5
timeout 600 python tools/spmm_bench.py products 48:48,104:104,128:256 MPH_SPMM_CTAITEMS=0,4,8,16 2>&1 | tee gpurun_out/r2p_spmm_products.txt
