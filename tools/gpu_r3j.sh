#!/bin/bash
# reddit SpMM: SM slices of the row-order chunked CSR (MPH_SPMM_SLICE=1) vs the hub-first items.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
run() { echo -n "$1 "; env $1 timeout 600 python tools/spmm_items_bench.py reddit 128:128,48:48 2>&1 | grep "ms per call" | sed 's/ ld=[0-9]*//;s/ ms per call//;s/split=1 chunk=default//' | tr '\n' ' '; echo; }
for rep in 1 2; do
  run MPH_SPMM_SLICE=0
  run MPH_SPMM_SLICE=1
  run "MPH_SPMM_SLICE=1 MPH_SPMM_CHUNK_EDGES=1010"
  run "MPH_SPMM_SLICE=1 MPH_SPMM_SLICE_TAIL=0.3"
  run "MPH_SPMM_SLICE=1 MPH_SPMM_SLICE_TAIL=0.03"
done
M=gpu__time_duration.sum,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active
for sl in 1 0; do
MPH_SPMM_SLICE=$sl timeout 900 ncu --metrics $M --clock-control none -k regex:k_spmm --launch-skip 10 --launch-count 4 --csv python tools/spmm_items_bench.py reddit 128:128,48:48 > gpurun_out/r3j_ncu_slice$sl.csv 2>/dev/null
done
echo ncu done
