#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo

for c in products reddit arxiv; do timeout 600 python tools/env_sweep.py $c MPH_GEMM_EPIBUFS=3,2,3,2 2>&1 | tail -8; done
