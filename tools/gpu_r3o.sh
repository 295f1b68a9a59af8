#!/bin/bash
# Products GEMM NT launches of one epoch after the epilogue fixes: duration, DRAM bytes, stall mix.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__pcsamp_warps_issue_stalled_long_scoreboard,smsp__pcsamp_warps_issue_stalled_wait,smsp__pcsamp_warps_issue_stalled_selected,smsp__pcsamp_warps_issue_stalled_branch_resolving,smsp__pcsamp_warps_issue_stalled_short_scoreboard,smsp__pcsamp_warps_issue_stalled_barrier,smsp__pcsamp_warps_issue_stalled_sleeping,smsp__pcsamp_warps_issue_stalled_lg_throttle,smsp__pcsamp_warps_issue_stalled_mio_throttle,smsp__pcsamp_warps_issue_stalled_math_pipe_throttle,smsp__pcsamp_warps_issue_stalled_no_instructions,smsp__pcsamp_warps_issue_stalled_misc,smsp__pcsamp_warps_issue_stalled_drain,smsp__pcsamp_warps_issue_stalled_membar
timeout 900 ncu --metrics $M --section WarpStateStats --clock-control none -k regex:k_gemm_nt -s 5 -c 5 --csv python tools/profile_step.py --config products --epochs 2 > gpurun_out/r3o_gemm.csv 2> gpurun_out/r3o.err; echo "ncu rc=$?"
