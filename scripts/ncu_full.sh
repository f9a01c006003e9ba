#!/bin/bash
# one ncu --set full capture of the step's main kernels (1 GPU; short run)
set -x
mkdir -p gpurun_out
K="regex:k_attn_fa|k_attn_seg|k_attn_tc|k_post_qkv|k_post_residual|k_post_gu|k_gemm_tc"
BB_PROF_ITERS=1 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k "$K" -c 14 \
  -o gpurun_out/prof_c2_full_${BB_DTYPE:-bf16x2} -f python scripts/profile_step.py > gpurun_out/ncu_full_${BB_DTYPE:-bf16x2}.log 2>&1
tail -3 gpurun_out/ncu_full_${BB_DTYPE:-bf16x2}.log
