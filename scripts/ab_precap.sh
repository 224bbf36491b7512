#!/bin/bash
# MFA cores: how many K / V ring pages to prefill before the PDL wait (the Q
# load queues behind them): libafdk_cur (whole rings) vs k4v0 / k2v0 / k1v1
cd "$(dirname "$0")/.."
export PYTHONPATH=$PWD
timeout 600 python -m pytest tests/test_mfa_fp8_gpu.py tests/test_mfa_decode_gpu.py -q -x 2>&1 | tail -1
for r in 1 2; do
  for lib in libafdk_cur.so libafdk_k4v0.so libafdk_k2v0.so libafdk_k1v1.so; do
    for cfg in "64 4096" "256 4096"; do
      echo "$lib $cfg: $(AFDK_LIB=$PWD/paper_2507_19427_b200/$lib timeout 120 python scripts/bench_attn_fp8.py $cfg 2>&1 | grep -v mtp | grep KV | sed 's/ of HBM peak//' | tr '\n' ' ')"
    done
  done
done
bash scripts/ab_layer_libs.sh libafdk_cur.so libafdk_k4v0.so libafdk_k2v0.so libafdk_k1v1.so
