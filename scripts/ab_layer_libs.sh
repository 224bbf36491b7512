#!/bin/bash
# A/B of whole libraries on the config-2 layer (bf16 / e4m3 KV) and the cores:
#   scripts/ab_layer_libs.sh libafdk.so libafdk_head.so ...
cd "$(dirname "$0")/.."
export PYTHONPATH=$PWD
for r in 1 2; do
  for lib in "$@"; do
    echo "$lib: $(AFDK_LIB=$PWD/paper_2507_19427_b200/$lib timeout 600 python bench.py --steps 20 --warmup 5 --no-moe --no-afd --no-long --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step']*1e3,1), 'us/layer core', round(d['roofline']['launch_ms']*1e3,1), 'fp8 layer', round(d['config2_fp8_kv']['layer_ms']*1e3,1), 'fp8 core', round(d['config2_fp8_kv']['core_ms']*1e3,1))")"
  done
done
for lib in "$@"; do
  echo "$lib B=256 e4m3: $(AFDK_LIB=$PWD/paper_2507_19427_b200/$lib timeout 600 python bench.py --steps 10 --warmup 3 --batch 256 --no-moe --no-afd --no-long --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step']*1e3,1), 'us/layer; e4m3', round(d['config2_fp8_kv']['layer_ms']*1e3,1))")"
done
