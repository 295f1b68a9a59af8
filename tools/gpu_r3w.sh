#!/bin/bash
# Next row's ids carried across contiguous rows (lib_x = in-tree) vs lib_c: kernel / e2e / hub-row
# tests, then per-call SpMM on products / reddit / arxiv, alternating.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
LIB=paper_2512_01678_b200/lib/libmorphling.so
cp $LIB /tmp/lib_cur.so
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_e2e.py tests/test_gpu_nell.py tests/test_gpu_fullsize.py -m gpu -q --timeout 1200 -p no:cacheprovider -k "spmm or sparse or e2e or nell or hub_rows or epoch" > gpurun_out/r3w_t.log 2>&1; echo "tests rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r3w_t.log | head -10
for rep in 1 2; do for lib in c x; do
  cp abtmp/lib_$lib.so $LIB
  echo -n "$lib "; timeout 600 python tools/spmm_items_bench.py products 256:256,104:104,48:48 2>&1 | grep "ms per call" | sed 's/ ld=[0-9]*//;s/ ms per call//;s/split=1 chunk=default//' | tr '\n' ' '; echo
  echo -n "$lib "; timeout 600 python tools/spmm_items_bench.py reddit 128:128,48:48 2>&1 | grep "ms per call" | sed 's/ ld=[0-9]*//;s/ ms per call//;s/split=1 chunk=default//' | tr '\n' ' '; echo
  echo -n "$lib "; timeout 600 python tools/spmm_items_bench.py arxiv 256:256,40:40 2>&1 | grep "ms per call" | sed 's/ ld=[0-9]*//;s/ ms per call//;s/split=1 chunk=default//' | tr '\n' ' '; echo
done; done
cp /tmp/lib_cur.so $LIB
