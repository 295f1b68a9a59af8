#!/bin/bash
# products 48-wide: row-slot kernel with 2 slots of 16 lanes (MPH_SPMM_ROWS=1 MPH_SPMM_ROWS16=1) vs k_spmm<16,1>.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
MPH_SPMM_ROWS=1 MPH_SPMM_ROWS16=1 timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "spmm_widths or row_slots or sign_bytes" > gpurun_out/r3p_t.log 2>&1; echo "tests rc=$?"
grep -E "passed|failed|FAILED" gpurun_out/r3p_t.log | head -5
run() { echo -n "$1 "; env $1 timeout 600 python tools/spmm_items_bench.py products 48:48 2>&1 | grep "ms per call" | sed 's/ ld=[0-9]*//;s/ ms per call//' | tr '\n' ' '; echo; }
for rep in 1 2 3; do
  run MPH_SPMM_ROWS=0
  run "MPH_SPMM_ROWS=1 MPH_SPMM_ROWS16=1"
done
