#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 600 python tools/spmm_bench.py reddit 48:48,64:128,128:128 MPH_SPMM_SMRANGE=0,1 2>&1 | tee gpurun_out/r2j_reddit.txt
timeout 600 python tools/spmm_bench.py products 48:48,104:104,128:256 MPH_SPMM_SMRANGE=0,1 2>&1 | tee gpurun_out/r2j_products.txt
timeout 600 python tools/env_sweep.py reddit MPH_SPMM_SMRANGE=0,1 2>&1 | tee gpurun_out/r2j_sweep_reddit.txt
timeout 600 python tools/env_sweep.py products MPH_SPMM_SMRANGE=0,1 2>&1 | tee gpurun_out/r2j_sweep_products.txt
