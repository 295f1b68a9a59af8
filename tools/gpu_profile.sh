#!/bin/bash
# ncu evidence: launch list of the bench command + --set full captures of the hot kernels
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
TAG=${1:-r01}
timeout 1200 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_bench.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --secondary none --no-probe > gpurun_out/${TAG}_launches_bench.out 2>&1; echo "launch list rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_spmm -s 4 -c 4 -o gpurun_out/${TAG}_spmm_reddit python tools/profile_step.py --config reddit --epochs 2 > /dev/null 2>&1; echo "spmm reddit rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_spmm -s 5 -c 5 -o gpurun_out/${TAG}_spmm_products python tools/profile_step.py --config products --epochs 2 > /dev/null 2>&1; echo "spmm products rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_gemm -s 8 -c 8 -o gpurun_out/${TAG}_gemm_products python tools/profile_step.py --config products --epochs 2 > /dev/null 2>&1; echo "gemm products rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_gemm -s 5 -c 5 -o gpurun_out/${TAG}_gemm_reddit python tools/profile_step.py --config reddit --epochs 2 > /dev/null 2>&1; echo "gemm reddit rc=$?"
ls -la gpurun_out/${TAG}_*
