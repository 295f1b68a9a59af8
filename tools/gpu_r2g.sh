#!/bin/bash
# round 2: degree-class L2 hints on products (correctness + A/B sweep)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -s --timeout 800 -p no:cacheprovider -k "degree_class" > gpurun_out/r2g_tests.log 2>&1; echo "gpu tests rc=$?"
grep -E "passed|failed|FAILED|Error|max \|err" gpurun_out/r2g_tests.log | head -20
timeout 900 python tools/env_sweep.py products MPH_SPMM_HOTMB=0,32,64,96 MPH_SPMM_L2POL=0,1,2,3 2>&1 | tee gpurun_out/r2g_sweep.txt | tail -32
