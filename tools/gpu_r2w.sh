#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 600 python tools/spmm_bench.py reddit 48:48,48:48b,64:128,64:128b,128:128,128:128b 2>&1
timeout 600 python tools/spmm_bench.py products 48:48,48:48b,128:256,128:256b 2>&1
