#!/bin/bash
# Round-2 evidence run (session 3 final code incl. the item-size changes): GPU parity suite + smoke, ncu launch list and --set full captures of the
# final code (-> profiles/r02_final8_*), DRAM traffic per aggregation call from those captures,
# then the default bench line (which reads that traffic) and the reference (oracle) arm.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
# (GPU suite: tools/gpu_r3z.sh, profiles/r02_final8_gpu_tests.txt)
bash tools/gpu_profile.sh r02_final8
python tools/traffic_from_ncu.py gpurun_out/r02_final8_ncu_full.json && cp profiles/ncu_traffic_*.json gpurun_out/
timeout 1200 python bench.py > gpurun_out/r02_final8_bench.json 2> gpurun_out/r02_final8_bench.err; echo "bench rc=$?"
# (reference arm: profiles/r02_final6_reference.json, the oracle is unchanged)
python - <<'PY'
import json
d = json.loads(open('gpurun_out/r02_final8_bench.json').read().strip().splitlines()[-1])
r = d['roofline']
print('bench', d['config']['workload'], round(d['value'], 3), 'e2e', round(d['e2e']['value'], 2), 'frac', round(r['frac'], 3),
      'dram_frac', r.get('dram_frac_of_hbm'), 'launches', d['gpu_launches'], 'clk', d['clocks'])
for n, s in (d.get('secondary') or {}).items(): print('  secondary', n, round(s['value'], 3))
ref = json.loads(open('gpurun_out/r02_final8_reference.json').read().strip().splitlines()[-1])
print('reference', ref.get('value'), ref.get('unit'), ref.get('cpu_baseline', {}).get('cores'))
PY
