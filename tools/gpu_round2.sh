#!/bin/bash
# tests + smoke + bench (reddit, arxiv, products, cora) + ncu launch list and full captures
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
bash tools/gpu_tests.sh
for c in reddit products arxiv pubmed; do
  timeout 900 python bench.py --config $c --steps 30 --warmup 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
done
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_reddit.csv python tools/profile_step.py --config reddit --epochs 2 > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_spmm -s 2 -c 4 -o gpurun_out/prof_spmm_reddit python tools/profile_step.py --config reddit --epochs 2 > gpurun_out/ncu_spmm.log 2>&1; echo "ncu spmm rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_gemm -s 0 -c 5 -o gpurun_out/prof_gemm_reddit python tools/profile_step.py --config reddit --epochs 1 > gpurun_out/ncu_gemm.log 2>&1; echo "ncu gemm rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_spmm -s 0 -c 3 -o gpurun_out/prof_spmm_products python tools/profile_step.py --config products --epochs 1 > gpurun_out/ncu_spmm_p.log 2>&1; echo "ncu spmm products rc=$?"
ls -la gpurun_out | head -40
