#!/bin/bash
# products: the one-slot row-slot kernel (next row's ids loaded during the current row's last step)
# for 104/128-wide rows on the chunked CSR (MPH_SPMM_ROWS_WIDE=1) vs k_spmm<32,1>; parity first.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
MPH_SPMM_ROWS_WIDE=1 timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "spmm" > gpurun_out/r3k_t.log 2>&1; echo "spmm tests (ROWS_WIDE=1) rc=$?"
grep -E "passed|failed|FAILED|Error|assert" gpurun_out/r3k_t.log | head -10
run() { echo -n "$1 "; env $1 timeout 600 python tools/spmm_items_bench.py products $2 2>&1 | grep "ms per call" | sed 's/ ld=[0-9]*//;s/ ms per call//;s/split=1 chunk=default//' | tr '\n' ' '; echo; }
for rep in 1 2 3; do
  run MPH_SPMM_ROWS_WIDE=0 256:256,104:104
  run MPH_SPMM_ROWS_WIDE=1 256:256,104:104
done
