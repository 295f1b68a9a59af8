#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
MPH_SPMM_WIDE=1 timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -s --timeout 800 -p no:cacheprovider -k "spmm" > gpurun_out/r2q_tests.log 2>&1; echo "gpu tests rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2q_tests.log | head -5
timeout 600 python tools/spmm_bench.py products 48:48,104:104,128:256 MPH_SPMM_WIDE=0,1,2,3 2>&1 | tee gpurun_out/r2q_spmm_products.txt
timeout 600 python tools/spmm_bench.py reddit 64:128 MPH_SPMM_WIDE=0,1,2,3 2>&1 | tee gpurun_out/r2q_spmm_reddit.txt
timeout 600 python tools/env_sweep.py products MPH_SPMM_WIDE=0,1,2,3 2>&1 | tee gpurun_out/r2q_sweep_products.txt
