#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
run() {
  local tag=$1; shift
  local cfg=$1; shift
  env "$@" timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-probe --secondary none > gpurun_out/sw_${tag}_${cfg}.json 2>/dev/null
  python - "$tag" "$cfg" <<'PY'
import json,sys
t,c=sys.argv[1],sys.argv[2]
try: d=json.load(open(f'gpurun_out/sw_{t}_{c}.json'))
except Exception as e: print(t,c,'fail'); sys.exit()
print(t, c, round(d['value'],3), 'ms; spmm', round(d['kernels']['spmm']['ms_per_epoch'],3), 'loss', d.get('final_loss'))
PY
}
run base products A=0
run slab128 products MPH_SPMM_SLAB=128
run slab64 products MPH_SPMM_SLAB=64
run slab128u8 products MPH_SPMM_SLAB=128 MPH_SPMM_U32=16
run base reddit A=0
run slab64 reddit MPH_SPMM_SLAB=64
run slab32 reddit MPH_SPMM_SLAB=32
