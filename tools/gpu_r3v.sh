#!/bin/bash
# k_spmm_combine: 8 chunk loads in flight and a 2x grid (lib_comb8 = in-tree) vs 4 (lib_comb4); ncu times + per-call SpMM.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
LIB=paper_2512_01678_b200/lib/libmorphling.so
cp $LIB /tmp/lib_cur.so
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -p no:cacheprovider -k chunked > gpurun_out/r3v_t.log 2>&1; echo "tests rc=$?"; grep -E "passed|failed" gpurun_out/r3v_t.log
for lib in comb4 comb8; do
  cp abtmp/lib_$lib.so $LIB
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_spmm_combine -c 6 --csv python tools/spmm_items_bench.py products 256:256,104:104 2>/dev/null | grep k_spmm_combine | awk -F'","' '{print $NF}' | tr '\n' ' '; echo " <- $lib combine ns"
done
for rep in 1 2; do for lib in comb4 comb8; do
  cp abtmp/lib_$lib.so $LIB
  echo -n "$lib "; timeout 600 python tools/spmm_items_bench.py products 256:256,104:104 2>&1 | grep "ms per call" | sed 's/ ld=[0-9]*//;s/ ms per call//;s/split=1 chunk=default//' | tr '\n' ' '; echo
done; done
cp /tmp/lib_cur.so $LIB
