#!/bin/bash
# A/B the attention core across library variants in one GPU session (alternating, 2 rounds)
for r in 1 2; do
for v in "" _bf16p; do
  lib=paper_2507_19427_b200/libafdk$v.so
  AFDK_LIB=$PWD/$lib timeout 120 python bench.py --steps 30 --warmup 5 --workload attn --no-cpu-baseline --no-moe --no-afd 2>/tmp/ab_err.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v'.ljust(10), round(d['roofline']['launch_ms']*1e3,2), 'us', round(d['roofline']['frac'],3))"
done; done; tail -3 /tmp/ab_err.log
