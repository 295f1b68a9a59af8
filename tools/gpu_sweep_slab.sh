#!/bin/bash
# SpMM column-slab policy check (MPH_SPMM_SLAB=-1 disables the default)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
run() {
  local tag=$1; shift
  local cfg=$1; shift
  env "$@" timeout 600 python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-probe --secondary none > gpurun_out/sw_${tag}_${cfg}.json 2>/dev/null
  python - "$tag" "$cfg" <<'PY'
import json,sys
t,c=sys.argv[1],sys.argv[2]
try: d=json.load(open(f'gpurun_out/sw_{t}_{c}.json'))
except Exception as e: print(t,c,'fail'); sys.exit()
print(t, c, round(d['value'],3), 'ms; spmm', round(d['kernels']['spmm']['ms_per_epoch'],3))
PY
}
for c in arxiv arxiv reddit; do
  run auto $c A=0
  run off $c MPH_SPMM_SLAB=-1
done
