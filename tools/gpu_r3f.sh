#!/bin/bash
# Chunked virtual CSR (in-tree = abtmp/lib_v4): SpMM tests, per-call SpMM head vs v4, epochs.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
LIB=paper_2512_01678_b200/lib/libmorphling.so
cp $LIB /tmp/lib_cur.so
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "spmm" > gpurun_out/r3f_t.log 2>&1; echo "spmm tests rc=$?"
grep -E "passed|failed|FAILED|Error|assert" gpurun_out/r3f_t.log | head -20
run() {  # lib split chunk cfg shapes
  cp abtmp/lib_$1.so $LIB
  if [ "$3" = d ]; then unset MPH_SPMM_CHUNK_EDGES; else export MPH_SPMM_CHUNK_EDGES=$3; fi
  echo -n "lib=$1 "; MPH_SPMM_SPLIT=$2 timeout 600 python tools/spmm_items_bench.py $4 $5 2>&1 | grep "ms per call" | sed 's/ ld=[0-9]*//;s/ ms per call//' | tr '\n' ' '; echo
}
for rep in 1 2; do
  run head 0 d products 256:256,104:104,48:48
  run v4 1 d products 256:256,104:104,48:48
  run v4 1 128 products 256:256,104:104,48:48
  run v4 0 d products 256:256,104:104,48:48
  run head 0 d reddit 128:128,48:48
  run v4 1 d reddit 128:128,48:48
  run v4 2 1010 reddit 128:128,48:48
  run head 0 d arxiv 256:256,40:40
  run v4 1 d arxiv 256:256,40:40
  run v4 0 d arxiv 256:256,40:40
done
unset MPH_SPMM_CHUNK_EDGES MPH_SPMM_SPLIT
cp /tmp/lib_cur.so $LIB
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
for cfg in products reddit arxiv; do
  timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-probe --secondary none > gpurun_out/r3f_$cfg.json 2> gpurun_out/r3f_$cfg.err
  echo -n "epoch v4: "; summ gpurun_out/r3f_$cfg.json
done
