#!/bin/bash
# Stall reasons / source hot spots of the products dH GEMM (K = 48, N = 256, sign-byte mask).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 ncu --section WarpStateStats --section SourceCounters --section SchedulerStats --clock-control none --import-source on \
  -k regex:k_gemm_nt -s 8 -c 1 -o gpurun_out/r3m_dh python tools/profile_step.py --config products --epochs 2 > gpurun_out/r3m.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/r3m_dh.ncu-rep --page raw --csv > gpurun_out/r3m_raw.csv 2>/dev/null
ncu -i gpurun_out/r3m_dh.ncu-rep --page source --csv --print-source sass > gpurun_out/r3m_src.csv 2>/dev/null
ncu -i gpurun_out/r3m_dh.ncu-rep --page details --csv > gpurun_out/r3m_details.csv 2>/dev/null
gzip -f gpurun_out/r3m_src.csv
rm -f gpurun_out/r3m_dh.ncu-rep
ls -la gpurun_out/r3m*
