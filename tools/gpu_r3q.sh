#!/bin/bash
# CUDA-graph replay of the epoch (bench.py --graph) vs eager launches, reddit and products, alternating.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
summ() {
python - "$1" <<'PY'
import json,sys
f=sys.argv[1]
try: d=json.loads(open(f).read().strip().splitlines()[-1])
except Exception as e: print(f,'no json', open(f.replace('.json','.err')).read()[-800:]); sys.exit()
print(d['config']['workload'], round(d['value'],3), d['config'].get('graph', d['config'].get('cuda_graph')), d.get('gpu_launches'))
PY
}
for rep in 1 2; do
  for cfg in reddit products; do
    for g in "" "--graph"; do
      timeout 600 python bench.py --config $cfg $g --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-probe --secondary none > gpurun_out/r3q.json 2> gpurun_out/r3q.err
      echo -n "$cfg $g: "; summ gpurun_out/r3q.json
    done
  done
done
