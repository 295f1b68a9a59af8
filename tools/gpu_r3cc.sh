#!/bin/bash
# Items of S/2 edges on the chunked CSR: chunked / hub / P2P-parts tests, products epochs.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fullsize.py tests/test_gpu_p2p.py tests/test_gpu_fullsize_train.py -m gpu -q --timeout 1200 -p no:cacheprovider -k "chunked or hub_rows or products" > gpurun_out/r3cc_t.log 2>&1; echo "tests rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r3cc_t.log | head -5
for rep in 1 2; do
  timeout 600 python bench.py --config products --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-probe --secondary none > gpurun_out/r3cc.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r3cc.json').read().strip().splitlines()[-1]);print('products',round(d['value'],3),{k:round(v['ms_per_epoch'],3) for k,v in d['kernels'].items()})"
done
