#!/bin/bash
# Round-2 sanitizer pass over the final kernels: memcheck over the single-process GPU tests,
# racecheck + synccheck + initcheck over the kernel tests (logs under gpurun_out/).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
bash tools/gpu_sanitize.sh
TOOLS="racecheck synccheck initcheck" bash tools/gpu_racecheck.sh
