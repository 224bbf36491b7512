#!/bin/bash
# compute-sanitizer passes over the small-shape GPU tests (memcheck, racecheck,
# synccheck); logs under gpurun_out/sanitizer_<tool>.log
set -u
CS=/usr/local/cuda/bin/compute-sanitizer
SEL='tests/test_mfa_decode_gpu.py::test_mfa_decode_parity tests/test_mfa_fp8_gpu.py tests/test_mfa_mtp_gpu.py tests/test_linear_gpu.py tests/test_moe_gpu.py::test_moe_ffn_small tests/test_moe_gpu.py::test_permute_bit_exact tests/test_moe_gpu.py::test_moe_ffn_many_rows_per_expert tests/test_moe_mx_gpu.py::test_moe_ffn_mx_small tests/test_moe_mx_gpu.py::test_moe_ffn_mx_two_accumulator_chunks tests/test_moe_bf16_gpu.py::test_moe_ffn_bf16_small tests/test_mfa_layer_gpu.py::test_mfa_layer_small_dims'
for tool in ${TOOLS:-memcheck racecheck synccheck}; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report hazard"
  timeout ${TMO:-900} $CS --tool $tool $extra --target-processes all --print-limit 50 \
    python -m pytest $SEL -q -x -p no:cacheprovider > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitizer_summary.txt
  grep -E "ERROR SUMMARY|passed|failed|Error" gpurun_out/sanitizer_$tool.log | tail -5 | tee -a gpurun_out/sanitizer_summary.txt
done
