#!/bin/bash
# Session-3 check of HEAD: GPU parity suite + smoke, default bench line, then the work-item size
# (MPH_SPMM_ITEM_EDGES) sweep on products / reddit (window of concurrently walked rows).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
bash tools/gpu_tests.sh
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r3a_bench.json 2> gpurun_out/r3a_bench.err; echo "bench rc=$?"
summ() {
python - "$1" <<'PY'
import json,sys
f=sys.argv[1]
try: d=json.loads(open(f).read().strip().splitlines()[-1])
except Exception as e: print(f,'no json'); sys.exit()
ks=' '.join(f"{k}={v['ms_per_epoch']:.3f}" for k,v in d['kernels'].items())
print(f, d['config']['workload'], round(d['value'],3), ks)
PY
}
summ gpurun_out/r3a_bench.json
for cfg in products reddit; do
  for ie in 0 1024 256 128 64; do
    if [ $ie = 0 ]; then unset MPH_SPMM_ITEM_EDGES; else export MPH_SPMM_ITEM_EDGES=$ie; fi
    timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-probe --secondary none > gpurun_out/r3a_${cfg}_ie$ie.json 2> gpurun_out/r3a_${cfg}_ie$ie.err
    echo -n "ie=$ie "; summ gpurun_out/r3a_${cfg}_ie$ie.json
  done
done
unset MPH_SPMM_ITEM_EDGES
