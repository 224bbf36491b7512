#!/bin/bash
# MFA cores: K pages of the next segment issued ahead of its Q (bf16) / bf16 Q
# released after quantisation + next Q quantised before the epilogue (e4m3):
# parity + A/B against libafdk_prevq.so (both off) and libafdk_q8only.so (e4m3 change only)
cd "$(dirname "$0")/.."
export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests/test_mfa_decode_gpu.py tests/test_mfa_fp8_gpu.py tests/test_mfa_layer_gpu.py \
  tests/test_bench_shapes_gpu.py tests/test_mfa_mtp_gpu.py -q -x 2>&1 | tail -2
for r in 1 2; do
  for lib in libafdk_cur.so libafdk_prevq.so libafdk_q8only.so; do
    for cfg in "64 4096" "32 32768" "256 4096" "320 4096"; do
      echo "$lib $cfg: $(AFDK_LIB=$PWD/paper_2507_19427_b200/$lib timeout 120 python scripts/bench_attn_fp8.py $cfg 2>&1 | grep -v mtp | tr '\n' ' ')"
    done
  done
done
bash scripts/ab_layer_libs.sh libafdk_cur.so libafdk_prevq.so
