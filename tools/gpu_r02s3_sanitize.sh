#!/bin/bash
# Round-2 session-3 sanitizer pass (chunked CSR, combine kernel, GEMM epilogue changes): memcheck over the single-process GPU tests,
# racecheck + synccheck + initcheck over the kernel tests (logs under gpurun_out/).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
bash tools/gpu_sanitize.sh
TOOLS="racecheck synccheck initcheck" bash tools/gpu_racecheck.sh
