#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 300 python tools/debug_tn.py > gpurun_out/debug_tn.log 2>&1
head -80 gpurun_out/debug_tn.log
