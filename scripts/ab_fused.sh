#!/bin/bash
# A/B: decode-batch MXFP8 MoE with the fused gate|up+down launch vs two launches
cd "$(dirname "$0")/.."
export PYTHONPATH=$PWD
for round in 1 2; do
  for f in 1 0; do
    for cfg in "256 1" "256 3" "256 6" "128 1" "64 3" "384 3"; do
      echo "fused=$f $(AFDK_MX_FUSED=$f timeout 120 python scripts/prof_moe_shard.py $cfg mx 2>&1 | tail -1)"
    done
  done
done
