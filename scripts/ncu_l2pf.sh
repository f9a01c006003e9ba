#!/bin/bash
# DRAM bytes per block-step GEMM with and without the next-GEMM L2 prefetch
# (single-pass metrics, caches not flushed between kernels)
mkdir -p gpurun_out
for mb in 0 48; do
  BB_L2PF_MB=$mb BB_PROF_ITERS=1 timeout 600 ncu --cache-control none --clock-control none \
    --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --profile-from-start off \
    -k regex:k_gemm_tc -c 12 --csv python scripts/profile_step.py > gpurun_out/ncu_l2pf_$mb.csv 2>&1
done
