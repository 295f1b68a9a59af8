#!/bin/bash
# arxiv (mean degree 7): ids carried across rows in the 128/256-wide warp-per-row launches
# (MPH_SPMM_CARRY_LOW=1) vs not; parity tests with it on.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
MPH_SPMM_CARRY_LOW=1 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_e2e.py -m gpu -q --timeout 600 -p no:cacheprovider -k "spmm or e2e or epoch" > gpurun_out/r3aa_t.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed" gpurun_out/r3aa_t.log | head -3
for rep in 1 2; do for v in 0 1; do
  if [ $v = 1 ]; then export MPH_SPMM_CARRY_LOW=1; else unset MPH_SPMM_CARRY_LOW; fi
  echo -n "carry_low=$v "; timeout 600 python tools/spmm_items_bench.py arxiv 256:256,128:128 2>&1 | grep "ms per call" | sed 's/ ld=[0-9]*//;s/ ms per call//;s/split=1 chunk=default//' | tr '\n' ' '; echo
  timeout 600 python bench.py --config arxiv --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-probe --secondary none > gpurun_out/r3aa.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r3aa.json').read().strip().splitlines()[-1]);print('   epoch',round(d['value'],4),{k:round(v['ms_per_epoch'],4) for k,v in d['kernels'].items()})"
done; done
