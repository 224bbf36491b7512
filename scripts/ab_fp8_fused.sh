#!/bin/bash
# FP8 (1x128) decode MoE: fused gate|up+down launch vs two launches; parity (1 GPU)
cd "$(dirname "$0")/.."
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_moe_gpu.py tests/test_bench_shapes_gpu.py tests/test_error_budget_gpu.py -q -x 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for r in 1 2; do
  for f in 1 0; do
    for cfg in "256 1" "256 3" "192 3" "64 3" "384 3"; do
      echo "fused=$f $(AFDK_FP8_FUSED=$f timeout 120 python scripts/prof_moe_shard.py $cfg fp8 2>&1 | tail -1)"
    done
  done
done
