#!/bin/bash
# Full GPU parity suite + smoke at the chunked-CSR code, then the products / arxiv / reddit epochs.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
bash tools/gpu_tests.sh
summ() {
python - "$1" <<'PY'
import json,sys
f=sys.argv[1]
try: d=json.loads(open(f).read().strip().splitlines()[-1])
except Exception as e: print(f,'no json'); sys.exit()
ks=' '.join(f"{k}={v['ms_per_epoch']:.3f}" for k,v in d['kernels'].items())
print(d['config']['workload'], round(d['value'],3), ks)
PY
}
for cfg in products arxiv reddit; do
  timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-probe --secondary none > gpurun_out/r3g_$cfg.json 2> gpurun_out/r3g_$cfg.err
  echo -n "epoch: "; summ gpurun_out/r3g_$cfg.json
done
