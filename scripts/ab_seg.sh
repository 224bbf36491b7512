#!/bin/bash
# A/B of the MFA segment charge (bf16 / e4m3 cores) and K3's poll back-off
cd "$(dirname "$0")/.."
export PYTHONPATH=$PWD
for round in 1 2; do
  for sc in 3 5 7 9; do
    echo "e4m3 seg_cost=$sc: $(AFDK_MFA8_SEG_COST=$sc timeout 120 python scripts/bench_attn_fp8.py 64 4096 2>&1 | grep '^e4m3')"
    echo "e4m3 seg_cost=$sc B256: $(AFDK_MFA8_SEG_COST=$sc timeout 120 python scripts/bench_attn_fp8.py 256 4096 2>&1 | grep '^e4m3')"
  done
  for sc in 2 3 4 6; do
    echo "bf16 seg_cost=$sc: $(AFDK_MFA_SEG_COST_RT=$sc timeout 120 python scripts/bench_attn_fp8.py 64 4096 2>&1 | grep '^bf16')"
  done
  echo "new: $(timeout 120 python scripts/bench_attn_fp8.py 64 4096 2>&1 | grep -v mtp)"
  for v in oldk3 k3s256; do
    echo "$v: $(AFDK_LIB=$PWD/paper_2507_19427_b200/libafdk_$v.so timeout 120 python scripts/bench_attn_fp8.py 64 4096 2>&1 | grep -v mtp)"
  done
done
