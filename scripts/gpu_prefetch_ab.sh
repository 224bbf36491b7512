#!/bin/bash
# MFA K/V ring prefill before the PDL wait: parity + A/B (1 GPU)
cd "$(dirname "$0")/.."
export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests/test_mfa_decode_gpu.py tests/test_mfa_fp8_gpu.py tests/test_mfa_layer_gpu.py \
  tests/test_bench_shapes_gpu.py tests/test_mfa_mtp_gpu.py -q -x 2>&1 | tail -2
for lib in libafdk.so libafdk_noprefetch.so; do
  for cfg in "64 4096" "32 32768"; do
    echo "$lib $cfg: $(AFDK_LIB=$PWD/paper_2507_19427_b200/$lib timeout 120 python scripts/bench_attn_fp8.py $cfg 2>&1 | grep -v mtp | tr '\n' ' ')"
  done
done
bash scripts/ab_layer_libs.sh libafdk.so libafdk_noprefetch.so
