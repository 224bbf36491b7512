#!/bin/bash
# attention layer at AFD micro-batch sizes (256/320/384 requests): timings + serialised launch list (1 GPU)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONPATH=$PWD
for B in 256 320 384; do
  echo "B=$B $(timeout 600 python bench.py --steps 10 --warmup 3 --batch $B --no-moe --no-afd --no-long --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step']*1e3,1), 'us/layer bf16; core', round(d['roofline']['launch_ms']*1e3,1), '; e4m3 layer', round(d['config2_fp8_kv']['layer_ms']*1e3,1), 'core', round(d['config2_fp8_kv']['core_ms']*1e3,1))")"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_B$B.csv \
    python bench.py --steps 2 --warmup 3 --batch $B --no-moe --no-afd --no-long --no-cpu-baseline > /dev/null 2>&1
done
