#!/bin/bash
# compute-sanitizer racecheck / synccheck (TOOLS="initcheck" etc. to choose) over the GEMM and SpMM kernel tests (shared-memory
# hazards, illegal barrier use).  Logs under gpurun_out/.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in ${TOOLS:-racecheck synccheck}; do
  timeout 1500 $CS --tool $tool --print-limit 20 --log-file gpurun_out/${tool}_%p.log \
    python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider --timeout 1400 \
    -k "${1:-gemm or softmax or spmm_widths or row_slots or chunked}" > gpurun_out/${tool}_pytest.log 2>&1
  echo "$tool rc=$?"; tail -1 gpurun_out/${tool}_pytest.log
  grep -h "ERROR SUMMARY\|RACECHECK SUMMARY\|hazard" gpurun_out/${tool}_*.log | sort | uniq -c | head -10
done
