#!/bin/bash
# round 2: 48-wide SpMM lane shapes x row stride; hub-block A/B (reddit epoch + SpMM)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 600 python tools/spmm_bench.py reddit 48:48,48:64,64:128,128:128 MPH_SPMM_SHAPE12=0,1,2,3 2>&1 | tee gpurun_out/r2i_reddit.txt
timeout 600 python tools/spmm_bench.py products 48:48,48:64 MPH_SPMM_SHAPE12=0,1,2,3 2>&1 | tee gpurun_out/r2i_products.txt
B="python bench.py --steps 20 --warmup 5 --secondary none --no-cpu-baseline --no-e2e --no-probe"
timeout 600 $B > gpurun_out/r2i_bench_hub256.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/r2i_bench_hub256.json').read().strip().splitlines()[-1]);print('hub256',d['value'],d['kernels']['spmm']['ms_per_epoch'])"
cp paper_2512_01678_b200/lib/libmorphling.so /tmp/lib_hub256.so
MPH_BUILD_DEFINES="-DMPH_HUB_BLOCK=(1LL<<40)" python paper_2512_01678_b200/build.py --force > /dev/null 2>&1; echo "alt build rc=$?"
timeout 600 $B > gpurun_out/r2i_bench_hubinf.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/r2i_bench_hubinf.json').read().strip().splitlines()[-1]);print('hubinf',d['value'],d['kernels']['spmm']['ms_per_epoch'])"
cp /tmp/lib_hub256.so paper_2512_01678_b200/lib/libmorphling.so
timeout 600 $B > gpurun_out/r2i_bench_hub256b.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/r2i_bench_hub256b.json').read().strip().splitlines()[-1]);print('hub256 again',d['value'],d['kernels']['spmm']['ms_per_epoch'])"
