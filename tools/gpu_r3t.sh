#!/bin/bash
# Layer-1 dW GEMM pipelined with the second slab of the last aggregation (lib_pipe = in-tree) vs
# lib_base: e2e / full-size training tests, then reddit / products epochs alternating.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
LIB=paper_2512_01678_b200/lib/libmorphling.so
cp $LIB /tmp/lib_cur.so
timeout 1500 python -m pytest tests/test_gpu_e2e.py tests/test_gpu_fullsize_train.py tests/test_gpu_boundary.py -m gpu -q --timeout 1200 -p no:cacheprovider > gpurun_out/r3t_t.log 2>&1; echo "tests rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r3t_t.log | head -10
for rep in 1 2 3; do
  for lib in base pipe; do
    cp abtmp/lib_$lib.so $LIB
    for cfg in reddit; do
      timeout 600 python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-probe --secondary none > gpurun_out/r3t.json 2> gpurun_out/r3t.err
      python -c "import json;d=json.loads(open('gpurun_out/r3t.json').read().strip().splitlines()[-1]);print('lib=$lib $cfg',round(d['value'],3),{k:(round(v['ms_per_epoch'],3),v['launches_per_epoch']) for k,v in d['kernels'].items()})"
    done
  done
done
cp /tmp/lib_cur.so $LIB
