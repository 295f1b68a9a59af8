#!/bin/bash
# Chunked virtual CSRs for the row parts (P > 1): P2P suite (incl. full size, and the forced-split
# cases), SpMM kernel tests, products / reddit epochs.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 1800 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_kernels.py -m gpu -q --timeout 900 -p no:cacheprovider -k "p2p or spmm or share" > gpurun_out/r3r_t.log 2>&1; echo "tests rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r3r_t.log | head -10
for cfg in products reddit; do
  timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-probe --secondary none > gpurun_out/r3r_$cfg.json 2> gpurun_out/r3r_$cfg.err
  python -c "import json;d=json.loads(open('gpurun_out/r3r_$cfg.json').read().strip().splitlines()[-1]);print('$cfg',round(d['value'],3),{k:round(v['ms_per_epoch'],3) for k,v in d['kernels'].items()})"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --share-device --comm p2p --config products --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-probe --secondary none > gpurun_out/r3r_share.json 2> gpurun_out/r3r_share.err; echo "share-device products rc=$?"; tail -c 400 gpurun_out/r3r_share.json
