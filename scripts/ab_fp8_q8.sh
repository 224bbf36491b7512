#!/bin/bash
# e4m3 core: next segment's Q quantised before the epilogue (double-buffered Q8) vs before: parity + A/B (1 GPU)
cd "$(dirname "$0")/.."
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_mfa_fp8_gpu.py tests/test_mfa_layer_gpu.py tests/test_bench_shapes_gpu.py -q -x 2>&1 | tail -2
for r in 1 2; do
  for lib in libafdk.so libafdk_prev.so; do
    for cfg in "64 4096" "32 32768" "256 4096" "320 4096"; do
      echo "$lib $cfg: $(AFDK_LIB=$PWD/paper_2507_19427_b200/$lib timeout 120 python scripts/bench_attn_fp8.py $cfg 2>&1 | grep '^e4m3')"
    done
  done
done
bash scripts/ab_layer_libs.sh libafdk.so libafdk_prev.so
