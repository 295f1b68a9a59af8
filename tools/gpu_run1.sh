#!/bin/bash
# First GPU pass: kernel parity, e2e parity, smoke, short bench.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
python -c "import torch; print(torch.cuda.get_device_name(0))" > gpurun_out/dev.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q --timeout 300 -p no:cacheprovider > gpurun_out/t_kernels.log 2>&1; echo "kernels rc=$?" >> gpurun_out/summary.txt
timeout 1200 python -m pytest tests/test_gpu_e2e.py -q --timeout 600 -p no:cacheprovider > gpurun_out/t_e2e.log 2>&1; echo "e2e rc=$?" >> gpurun_out/summary.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/summary.txt
timeout 600 python bench.py --config arxiv --steps 20 --warmup 5 > gpurun_out/bench_arxiv.log 2>&1; echo "bench arxiv rc=$?" >> gpurun_out/summary.txt
timeout 900 python bench.py --config reddit --steps 20 --warmup 5 > gpurun_out/bench_reddit.log 2>&1; echo "bench reddit rc=$?" >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
tail -5 gpurun_out/t_kernels.log
