#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider -k "graph or adam or dropout or loss_traj" > gpurun_out/t_quick.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_quick.log
for c in cora pubmed arxiv; do
 for gflag in "" "--graph"; do
  timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --secondary none --no-probe $gflag > gpurun_out/bg.json 2> gpurun_out/bg.err; echo "bench $c $gflag rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/bg.json')); print('  ', d['config']['workload'], d['config']['cuda_graph'], round(d['value'],4), 'ms/epoch; e2e', round(d['e2e']['value'],3))" || tail -3 gpurun_out/bg.err
 done
done
