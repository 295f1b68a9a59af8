#!/bin/bash
# products 48-wide SpMM: chunked CSR vs hub-first items, alternating processes.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
run() { echo -n "$1 "; env $1 timeout 600 python tools/spmm_items_bench.py products $2 2>&1 | grep "ms per call" | sed 's/ ld=[0-9]*//;s/ ms per call//' | tr '\n' ' '; echo; }
for rep in 1 2 3; do
  run MPH_SPMM_SPLIT=0 48:48,104:104
  run MPH_SPMM_SPLIT=1 48:48,104:104
done
