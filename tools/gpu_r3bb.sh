#!/bin/bash
# products chunked CSR: edges per work item (MPH_SPMM_RUN_EDGES) at chunk size 256.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for rep in 1 2; do for r in 0 32 64 96 128; do
  if [ $r = 0 ]; then unset MPH_SPMM_RUN_EDGES; else export MPH_SPMM_RUN_EDGES=$r; fi
  echo -n "run=$r "; timeout 600 python tools/spmm_items_bench.py products 256:256,104:104 2>&1 | grep "ms per call" | sed 's/ ld=[0-9]*//;s/ ms per call//;s/split=1 chunk=default//' | tr '\n' ' '; echo
done; done
