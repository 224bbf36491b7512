#!/bin/bash
# K3 batched merge + segment charge A/B, dense fused A/B (1 GPU)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_mfa_decode_gpu.py tests/test_mfa_fp8_gpu.py tests/test_mfa_mtp_gpu.py tests/test_mfa_layer_gpu.py -q -x 2>&1 | tail -3
AFDK_DENSE_FUSED=1 timeout 600 python -m pytest tests/test_moe_mx_gpu.py -q -x -k dense 2>&1 | tail -3
for r in 1 2; do
  for f in 1 0; do AFDK_DENSE_FUSED=$f timeout 300 python scripts/ab_dense_fused.py 2>&1 | grep '^{'; done
done
bash scripts/ab_seg.sh 2>&1
