#!/bin/bash
# compute-sanitizer memcheck over the single-process GPU tests (out-of-bounds / misaligned device
# accesses).  Skipped: full-size cases (time), the multi-process P2P cases, and the allocator test
# (under the sanitizer the frames of finished library calls stay referenced, so its "every
# allocation released on del" check cannot hold; it passes without the sanitizer).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 2400 $CS --tool memcheck --print-limit 20 --error-exitcode 9 --log-file gpurun_out/sanitize_%p.log \
  python -m pytest tests/test_gpu_kernels.py tests/test_gpu_boundary.py tests/test_gpu_aggregators.py \
  tests/test_gpu_bf16.py tests/test_gpu_e2e.py tests/test_gpu_nell.py -m gpu -q \
  --timeout 2000 -p no:cacheprovider -k "${1:-not fullsize and not set_allocator_torch and not full_size}" > gpurun_out/sanitize_pytest.log 2>&1
echo "memcheck rc=$?"
tail -3 gpurun_out/sanitize_pytest.log
grep -h "ERROR SUMMARY\|Invalid\|misaligned\|out of bounds" gpurun_out/sanitize_*.log | sort | uniq -c | head -20
