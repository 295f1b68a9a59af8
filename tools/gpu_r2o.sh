#!/bin/bash
# round 2: CTA-shared item scheduling — parity with the knob on, and A/B
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
MPH_SPMM_CTAITEMS=1 timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -s --timeout 800 -p no:cacheprovider -k "spmm" > gpurun_out/r2o_tests.log 2>&1; echo "gpu tests rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2o_tests.log | head -20
timeout 600 python tools/spmm_bench.py products 48:48,104:104,128:256 MPH_SPMM_CTAITEMS=0,1 2>&1 | tee gpurun_out/r2o_spmm_products.txt
timeout 600 python tools/spmm_bench.py reddit 48:48,64:128 MPH_SPMM_CTAITEMS=0,1 2>&1 | tee gpurun_out/r2o_spmm_reddit.txt
for c in products reddit; do timeout 600 python tools/env_sweep.py $c MPH_SPMM_CTAITEMS=0,1 2>&1 | tee gpurun_out/r2o_sweep_$c.txt; done
