#!/bin/bash
# dH GEMM without the fallback mask load + STS/LDS epilogue staging (lib_h = in-tree) vs lib_c (before the session-3 GEMM changes)
# vs the committed code (lib_c): GEMM / SpMM kernel tests, then epochs, alternating.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
LIB=paper_2512_01678_b200/lib/libmorphling.so
cp $LIB /tmp/lib_cur.so
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_bf16.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "gemm or sign or bf16" > gpurun_out/r3n_t.log 2>&1; echo "tests rc=$?"
grep -E "passed|failed|FAILED|Error|assert" gpurun_out/r3n_t.log | head -10
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
for rep in 1 2; do
  for lib in c h; do
    cp abtmp/lib_$lib.so $LIB
    for cfg in products products:bf16 reddit arxiv; do
      c=${cfg%%:*}; pr=tf32; [ "$cfg" != "$c" ] && pr=bf16
      timeout 600 python bench.py --config $c --precision $pr --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-probe --secondary none > gpurun_out/r3n_$lib.json 2> gpurun_out/r3n_$lib.err
      echo -n "lib=$lib $pr "; summ gpurun_out/r3n_$lib.json
    done
  done
done
cp /tmp/lib_cur.so $LIB
