#!/bin/bash
# A/B of prebuilt libraries (abtmp/lib_<name>.so swapped in place) x MPH_SPMM_SPLIT on products/reddit/arxiv.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
LIB=paper_2512_01678_b200/lib/libmorphling.so
cp $LIB /tmp/lib_cur.so
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "spmm" > gpurun_out/r3c_t.log 2>&1; echo "spmm tests (in-tree lib) rc=$?"
grep -E "passed|failed|FAILED|Error|assert" gpurun_out/r3c_t.log | head -20
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
  for v in ${VARIANTS:-head:0 noinl:1 noinl:0 inline:1 head:0 noinl:1}; do
    lib=${v%%:*}; sp=${v##*:}
    cp abtmp/lib_$lib.so $LIB
    export MPH_SPMM_SPLIT=$sp
    timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-probe --secondary none > gpurun_out/r3c_${cfg}_${lib}_$sp.json 2> gpurun_out/r3c_${cfg}_${lib}_$sp.err
    echo -n "lib=$lib split=$sp "; summ gpurun_out/r3c_${cfg}_${lib}_$sp.json
  done
done
cp /tmp/lib_cur.so $LIB
