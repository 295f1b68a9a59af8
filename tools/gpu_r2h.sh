#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python tools/env_sweep.py products MPH_SPMM_PERSIST_MB=0,64,96 MPH_SPMM_HOTMB=0,64 MPH_SPMM_L2POL=1,3 2>&1 | tee gpurun_out/r2h_sweep.txt | tail -24
