#!/bin/bash
# Hub-first items: edges per item E (MPH_SPMM_ITEM_EDGES; default nnz/(148*24*32) clamped: products
# 566, reddit 1010) for the launches that keep them (products 48-wide, reddit).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for rep in 1 2; do for ie in 0 512 256; do
  if [ $ie = 0 ]; then unset MPH_SPMM_ITEM_EDGES; else export MPH_SPMM_ITEM_EDGES=$ie; fi
  echo -n "E=$ie "; timeout 600 python tools/spmm_items_bench.py products 48:48 2>&1 | grep "ms per call" | sed 's/ ld=[0-9]*//;s/ ms per call//;s/split=1 chunk=default//' | tr '\n' ' '
  timeout 600 python tools/spmm_items_bench.py reddit 128:128,48:48 2>&1 | grep "ms per call" | sed 's/ ld=[0-9]*//;s/ ms per call//;s/split=1 chunk=default//' | tr '\n' ' '; echo
done; done
