#!/bin/bash
# router GEMM with the tokens as the M panels (tiles = token blocks) vs the gate rows as M: parity + A/B (1 GPU)
cd "$(dirname "$0")/.."
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_moe_gpu.py tests/test_moe_mx_gpu.py tests/test_moe_bf16_gpu.py tests/test_bench_shapes_gpu.py -q -x 2>&1 | tail -2
for lib in libafdk.so libafdk_oldrouter.so; do
  echo "$lib: $(AFDK_LIB=$PWD/paper_2507_19427_b200/$lib timeout 300 python scripts/prof_router.py 2>&1 | tr '\n' ' ')"
  for t in 368 256; do
    echo "$lib: $(AFDK_LIB=$PWD/paper_2507_19427_b200/$lib timeout 400 python scripts/afd_attn_breakdown.py $t 2>&1 | tail -2 | tr '\n' ' ')"
  done
done
