#!/bin/bash
# Per-call SpMM times of prebuilt libraries x MPH_SPMM_SPLIT (tools/spmm_items_bench.py), then ncu
# DRAM bytes / L2 hit rate of the products launches with and without chunked items.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
LIB=paper_2512_01678_b200/lib/libmorphling.so
cp $LIB /tmp/lib_cur.so
for v in head:0 noinl:0 noinl:1 head:0 noinl:1; do
  lib=${v%%:*}; sp=${v##*:}
  cp abtmp/lib_$lib.so $LIB
  echo "== lib=$lib"
  MPH_SPMM_SPLIT=$sp timeout 600 python tools/spmm_items_bench.py products 256:256,104:104,48:48 2>&1 | grep "ms per call"
  MPH_SPMM_SPLIT=$sp timeout 600 python tools/spmm_items_bench.py reddit 128:128,48:48 2>&1 | grep "ms per call"
done
cp abtmp/lib_noinl.so $LIB
for sp in 0 1; do
  MPH_SPMM_SPLIT=$sp timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_spmm --launch-skip 10 --launch-count 6 --csv python tools/spmm_items_bench.py products 256:256,104:104,48:48 > gpurun_out/r3d_ncu_products_split$sp.csv 2> gpurun_out/r3d_ncu_products_split$sp.err
  echo "ncu split=$sp rc=$?"
done
cp /tmp/lib_cur.so $LIB
