#!/bin/bash
# round 2: TMA gather4 SpMM — parity with the knob on, and A/B on products / reddit
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
MPH_SPMM_G4=1 timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -s --timeout 300 -p no:cacheprovider -k "spmm" > gpurun_out/r2r_tests.log 2>&1; echo "gpu tests rc=$?"
grep -E "passed|failed|FAILED|Error|error" gpurun_out/r2r_tests.log | head -8
timeout 300 python tools/spmm_bench.py products 48:48,128:256 MPH_SPMM_G4=0,1 2>&1 | tee gpurun_out/r2r_spmm_products.txt
timeout 300 python tools/spmm_bench.py reddit 64:128 MPH_SPMM_G4=0,1 2>&1 | tee gpurun_out/r2r_spmm_reddit.txt
