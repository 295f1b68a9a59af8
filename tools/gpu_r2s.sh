#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
MPH_SPMM_G4=1 timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none -k regex:k_spmm_g4 -s 2 -c 1 -o gpurun_out/r2s_g4 python tools/spmm_bench.py reddit 64:128 > gpurun_out/r2s.log 2>&1; echo "ncu rc=$?"
/usr/local/cuda/bin/ncu -i gpurun_out/r2s_g4.ncu-rep --page details --csv > gpurun_out/r2s_g4_details.csv 2>/dev/null
/usr/local/cuda/bin/ncu -i gpurun_out/r2s_g4.ncu-rep --page raw --csv > gpurun_out/r2s_g4_raw.csv 2>/dev/null
rm -f gpurun_out/r2s_g4.ncu-rep
