#!/bin/bash
# N=1 bench refresh (1-GPU box, like the driver's) + the reference arm
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/bench_n1_refresh.json 2> gpurun_out/bench_n1_refresh.err
tail -c 300 gpurun_out/bench_n1_refresh.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_refresh.json 2> gpurun_out/bench_ref_refresh.err
tail -c 400 gpurun_out/bench_ref_refresh.json
