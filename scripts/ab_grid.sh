#!/bin/bash
# A/B of the MFA decode core's CTA count at config 2 (core and layer), 2 alternating rounds
for r in 1 2; do
  for G in 148 128 136 144; do
    v=$(AFDK_MFA_GRID=$G timeout 300 python bench.py --workload attn --steps 30 --warmup 5 --no-moe --no-afd --no-long --no-cpu-baseline --no-fp8kv 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(round(d['roofline']['launch_ms']*1e3,2), round(d['roofline']['frac'],3))")
    l=$(AFDK_MFA_GRID=$G timeout 300 python bench.py --steps 20 --warmup 5 --no-moe --no-afd --no-long --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(round(d['ms_per_step']*1e3,2), round(d['layer_roofline']['frac'],3), round(d['config2_fp8_kv']['core_ms']*1e3,2))")
    echo "round $r G=$G core(us,frac)=$v layer(us,frac,fp8core)=$l"
  done
done
