#!/bin/bash
# round 2: row-block cache SpMM — parity (kernel tests + full reddit hubs) and A/B
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -m gpu -q -s --timeout 800 -p no:cacheprovider -k "spmm or hub or reddit_graph" > gpurun_out/r2m_tests.log 2>&1; echo "gpu tests rc=$?"
grep -E "passed|failed|FAILED|Error|max \|err" gpurun_out/r2m_tests.log | head -20
timeout 600 python tools/spmm_bench.py reddit 48:48,64:128,128:128 MPH_SPMM_CACHE=0,1 2>&1 | tee gpurun_out/r2m_spmm.txt
timeout 600 python tools/env_sweep.py reddit MPH_SPMM_CACHE=0,1 2>&1 | tee gpurun_out/r2m_sweep.txt
