#!/bin/bash
# A/B the e4m3-KV core's K/V ring depths across library variants (alternating, 2 rounds)
for r in 1 2; do
for v in "" _k4v5 _k3v6 _k2v4; do
  for shape in "64 4096" "32 32768"; do
    AFDK_LIB=$PWD/paper_2507_19427_b200/libafdk$v.so timeout 120 python scripts/bench_attn_fp8.py $shape 2>/tmp/ab_err.log | grep e4m3 | sed "s/^/${v:-base} /"
  done
done; done; tail -3 /tmp/ab_err.log
