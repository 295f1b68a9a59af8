#!/bin/bash
# Chunked items with the combine kernel (lib_v3 = in-tree): SpMM tests, then per-call SpMM times
# head vs v3 across MPH_SPMM_SPLIT / MPH_SPMM_CHUNK_EDGES.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
LIB=paper_2512_01678_b200/lib/libmorphling.so
cp $LIB /tmp/lib_cur.so
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "spmm" > gpurun_out/r3e_t.log 2>&1; echo "spmm tests rc=$?"
grep -E "passed|failed|FAILED|Error|assert" gpurun_out/r3e_t.log | head -20
run() {  # lib split chunk cfg shapes
  cp abtmp/lib_$1.so $LIB
  if [ "$3" = d ]; then unset MPH_SPMM_CHUNK_EDGES; else export MPH_SPMM_CHUNK_EDGES=$3; fi
  echo -n "lib=$1 "; MPH_SPMM_SPLIT=$2 timeout 600 python tools/spmm_items_bench.py $4 $5 2>&1 | grep "ms per call" | tr '\n' ' '; echo
}
for rep in 1 2; do
  run head 0 d products 256:256,104:104,48:48
  run v3 1 d products 256:256,104:104,48:48
  run v3 1 128 products 256:256,104:104,48:48
  run v3 1 512 products 256:256,104:104,48:48
  run v3 0 d products 256:256,104:104,48:48
done
for rep in 1 2; do
  run head 0 d reddit 128:128,48:48
  run v3 1 256 reddit 128:128,48:48
  run v3 1 1010 reddit 128:128,48:48
  run v3 1 2048 reddit 128:128,48:48
  run v3 0 d reddit 128:128,48:48
done
for rep in 1 2; do
  run head 0 d arxiv 256:256,40:40
  run v3 1 d arxiv 256:256,40:40
  run v3 1 256 arxiv 256:256,40:40
  run v3 0 d arxiv 256:256,40:40
done
cp /tmp/lib_cur.so $LIB
