#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider -k "${1:-softmax or probe}" > gpurun_out/t_quick.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_quick.log
timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_default.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench_default.json'))
print('main', d['config']['workload'], round(d['value'],3), 'e2e', round(d['e2e']['value'],2), 'cpu', round(d['cpu_baseline']['value']), 'launches', d['gpu_launches'], 'clk', d['clocks'])
print(' roofline', {k: (round(v,3) if isinstance(v,float) else v) for k,v in d['roofline'].items()})
for k,v in d['kernels'].items(): print('   ',k, round(v['ms_per_epoch'],3), 'ms', v['launches_per_epoch'], round(v['algorithmic_GBps']), 'GB/s')
for n,r in (d.get('secondary') or {}).items():
    print('secondary', n, round(r['value'],3), 'roofline frac', round(r['roofline']['frac'],3))
    for k,v in r['kernels'].items(): print('   ',k, round(v['ms_per_epoch'],3), 'ms', v['launches_per_epoch'], round(v['algorithmic_GBps']), 'GB/s')
PY
