#!/bin/bash
# Row-order items with chunked long rows: SpMM parity tests, then the A/B of
# MPH_SPMM_SPLIT (0: hub-first whole-row items) and the chunk size MPH_SPMM_CHUNK_EDGES.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "spmm" > gpurun_out/r3b_t.log 2>&1; echo "spmm tests rc=$?"
grep -E "passed|failed|FAILED|Error|assert" gpurun_out/r3b_t.log | head -20
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
for cfg in ${CFGS:-products reddit arxiv}; do
  for v in "0 0" "1 0" "1 128" "1 512" "0 0" "1 0"; do
    set -- $v
    export MPH_SPMM_SPLIT=$1
    if [ $2 = 0 ]; then unset MPH_SPMM_CHUNK_EDGES; else export MPH_SPMM_CHUNK_EDGES=$2; fi
    timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-probe --secondary none > gpurun_out/r3b_${cfg}_$1_$2.json 2> gpurun_out/r3b_${cfg}_$1_$2.err
    echo -n "split=$1 chunk=$2 "; summ gpurun_out/r3b_${cfg}_$1_$2.json
  done
done
