#!/bin/bash
# quick loop: selected tests + benches (args: pytest -k expr, configs)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
K=${1:-spmm}
shift
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider -k "$K" > gpurun_out/t_quick.log 2>&1; echo "tests rc=$?"
grep -E "passed|failed|FAILED|Error|assert" gpurun_out/t_quick.log | head -20
for c in "$@"; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bq_$c.json 2> gpurun_out/bq_$c.err; echo "bench $c rc=$?"
  python - "$c" <<'PY'
import json,sys
c=sys.argv[1]
try:
    d=json.load(open(f'gpurun_out/bq_{c}.json'))
except Exception as e:
    print(c, 'no json', open(f'gpurun_out/bq_{c}.err').read()[-2000:]); sys.exit()
print(c, round(d['value'],3), 'ms/epoch e2e', round(d['e2e']['value'],2), 'frac', round(d['roofline']['frac'],3), d['roofline']['kernel'])
for k,v in d['kernels'].items(): print('   ',k, round(v['ms_per_epoch'],3), 'ms', v['launches_per_epoch'], 'launches', round(v['algorithmic_GBps']), 'GB/s')
PY
done
