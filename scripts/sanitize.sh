#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck) over small GPU tests that
# exercise every kernel family: control + SIMT forward (fp32 full runs), the
# tcgen05 GEMMs, LM head and both tcgen05 attentions (bf16 / bf16x2 block
# steps at head_dim 128).  Logs -> gpurun_out/sanitizer_<tool>.txt
cd "$(dirname "$0")/.."
TESTS='tests/test_gpu_parity.py::test_fp32_matches_reference_runs[c1_hs2] tests/test_gpu_parity.py::test_block_step_hd128_attention_matches_oracle tests/test_gpu_parity.py::test_bf16x2_block_step_matches_exact_oracle tests/test_gpu_gemm.py'
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
    python -m pytest $TESTS -x -q -p no:cacheprovider > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "exit=$?" >> gpurun_out/sanitizer_$tool.txt
done
