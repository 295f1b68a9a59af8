#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
bash tools/gpu_quick.sh "spmm or e2e or fullsize" reddit products arxiv cora
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_spmm -s 2 -c 4 -o gpurun_out/prof_spmm_reddit_v3 python tools/profile_step.py --config reddit --epochs 2 > gpurun_out/ncu_spmm.log 2>&1; echo "ncu spmm rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_spmm -s 0 -c 5 -o gpurun_out/prof_spmm_products_v3 python tools/profile_step.py --config products --epochs 1 > gpurun_out/ncu_spmm_p.log 2>&1; echo "ncu spmm products rc=$?"
