#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 300 python tools/spmm_bench.py reddit 64:128 MPH_SPMM_G4=0,1,2 2>&1
timeout 300 python tools/spmm_bench.py products 128:256 MPH_SPMM_G4=0,1,2 2>&1
