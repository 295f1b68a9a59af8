#!/bin/bash
# products SpMM on the chunked CSR: column-slab width (MPH_SPMM_SLAB) and the row-slot kernel for 48-wide rows.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
run() { echo -n "$1 "; env $1 timeout 600 python tools/spmm_items_bench.py products $2 2>&1 | grep "ms per call" | sed 's/ ld=[0-9]*//;s/ ms per call//;s/split=1 chunk=default//' | tr '\n' ' '; echo; }
for rep in 1 2; do
  run MPH_SPMM_SLAB=0 256:256,48:48
  run MPH_SPMM_SLAB=-1 256:256
  run MPH_SPMM_SLAB=64 256:256
  run MPH_SPMM_ROWS=1 48:48
  run MPH_SPMM_SPLIT=0 48:48
done
