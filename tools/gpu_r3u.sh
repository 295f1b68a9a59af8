#!/bin/bash
# Full-size products hub-row SpMM parity (chunked CSR) test.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -s --timeout 1200 -p no:cacheprovider -k "hub_rows" > gpurun_out/r3u_t.log 2>&1; echo "tests rc=$?"
grep -E "passed|failed|FAILED|Error|max \|err\||assert" gpurun_out/r3u_t.log | head -20
