#!/bin/bash
# Full GPU parity suite + smoke at HEAD (after the chunked parts), then the default bench line.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
bash tools/gpu_tests.sh
timeout 1200 python bench.py > gpurun_out/r3ee_bench.json 2> gpurun_out/r3ee_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open('gpurun_out/r3ee_bench.json').read().strip().splitlines()[-1])
print('bench', d['config']['workload'], round(d['value'], 3), 'e2e', round(d['e2e']['value'], 2), 'frac', round(d['roofline']['frac'], 3), 'clk', d['clocks'])
for n, s in (d.get('secondary') or {}).items(): print('  secondary', n, round(s['value'], 3))
PY
