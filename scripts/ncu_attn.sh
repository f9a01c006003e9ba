#!/bin/bash
# ncu --set full of one block-pass attention launch, fused-QKV (FQ) vs separate finalize
mkdir -p gpurun_out
for v in 0 1; do
  BB_FQ=$((1-v)) BB_PROF_ITERS=1 timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:k_attn_seg -s 3 -c 1 -o gpurun_out/prof_attn_fq$((1-v)) -f python scripts/profile_step.py > gpurun_out/ncu_attn_$v.log 2>&1
  tail -2 gpurun_out/ncu_attn_$v.log
done
