#!/bin/bash
# compute-sanitizer (memcheck / synccheck / racecheck) over small GPU tests that
# exercise the product-path kernel families: control + SIMT forward (fp32
# full runs), the tcgen05 GEMMs + LM head, and the warp-specialized tcgen05
# attentions (64- and 128-row tiles, bf16 and bf16x2).  Logs ->
# gpurun_out/sanitizer_<tool>.txt
cd "$(dirname "$0")/.."
T=tests/test_gpu_parity.py
IDS="$T::test_fp32_matches_reference_runs[c1_hs2] tests/test_gpu_gemm.py::test_tc_gemm_partials[4096-4096-56-64]
 tests/test_gpu_gemm.py::test_tc_gemm_head_epilogue[4097-256-56-64]
 $T::test_block_step_hd128_attention_matches_oracle[fa--2-0.0-0.02]
 $T::test_block_step_hd128_attention_matches_oracle[fa64--2-0.0-0.02]
 $T::test_block_step_long_context_attention_matches_oracle[fa--600-200-4]
 $T::test_bf16x2_block_step_matches_exact_oracle[2-33.0-0.02-32-64]"
for tool in memcheck synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
    python -m pytest $IDS -q -p no:cacheprovider > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "exit=$?" >> gpurun_out/sanitizer_$tool.txt
done
