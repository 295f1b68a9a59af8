#!/bin/bash
# ncu evidence: launch list of the bench command + --set full captures of the hot kernels
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
TAG=${1:-r01}
timeout 1200 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_bench.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --secondary none --no-probe > gpurun_out/${TAG}_launches_bench.out 2>&1; echo "launch list rc=$?"
cap() {  # name regex skip count config [agg] [precision]
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$2 -s $3 -c $4 -o gpurun_out/${TAG}_$1 \
    python tools/profile_step.py --config $5 --epochs 2 --agg ${6:-gcn} --precision ${7:-tf32} > /dev/null 2>&1; echo "$1 rc=$?"
}
cap spmm_reddit k_spmm 6 6 reddit
cap spmm_products k_spmm 12 12 products   # 7 k_spmm + 5 k_spmm_combine per epoch (chunked CSR)
cap gemm_products k_gemm 8 8 products
cap gemm_reddit k_gemm 5 5 reddit
cap sparse_nell "k_spmm|k_sparse" 9 9 nell
cap aggmax_arxiv "k_aggmax|k_colsum" 7 6 arxiv max
cap gemm_products_bf16 k_gemm 8 8 products gcn bf16
# summaries on the box (the reports are too large to bring back: gpurun_out <= 64 MiB)
python tools/ncu_summary.py --launches gpurun_out/${TAG}_launches_bench.csv --out gpurun_out/${TAG}_launches_bench.md \
  --title "Launch list of python bench.py --steps 3 --warmup 3 (ncu --metrics gpu__time_duration.sum, cold, serialised)" > /dev/null
python tools/ncu_summary.py gpurun_out/${TAG}_*.ncu-rep --out gpurun_out/${TAG}_ncu_full.md --json gpurun_out/${TAG}_ncu_full.json \
  --title "ncu --set full --clock-control none captures (${TAG})" > /dev/null
for r in gpurun_out/${TAG}_*.ncu-rep; do
  ncu -i $r --page details --csv > ${r%.ncu-rep}_details.csv 2>/dev/null
  gzip -9 -f ${r%.ncu-rep}_details.csv
done
rm -f gpurun_out/${TAG}_*.ncu-rep
ls -la gpurun_out/${TAG}_*
