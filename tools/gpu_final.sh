#!/bin/bash
# Round-end check: the whole GPU parity suite + smoke, the default bench line and the reference
# (CPU oracle) arm, as the driver runs them.  Logs and JSON under gpurun_out/.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
bash tools/gpu_tests.sh
timeout 1200 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo "ref rc=$?"
python - <<'PY'
import json
d = json.load(open('gpurun_out/final_bench.json'))
print('bench', d['config']['workload'], round(d['value'], 3), 'e2e', round(d['e2e']['value'], 2), 'frac',
      round(d['roofline']['frac'], 3), 'launches', d['gpu_launches'], 'clk', d['clocks'])
for n, r in (d.get('secondary') or {}).items(): print('  secondary', n, round(r['value'], 3))
r = json.load(open('gpurun_out/final_ref.json'))
print('reference', r.get('value'), r.get('unit'), r.get('cpu_baseline', {}).get('sample'))
PY
