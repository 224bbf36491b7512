#!/bin/bash
# round-2 N=1: default bench, reference arm, launch list, one ncu --set full capture of the MFA core
set -u
mkdir -p gpurun_out
( time timeout 1200 python bench.py > gpurun_out/bench_n1_r02.json 2> gpurun_out/bench_n1_r02.err ) 2> gpurun_out/bench_n1_r02.time
tail -c 400 gpurun_out/bench_n1_r02.err; cat gpurun_out/bench_n1_r02.time
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r02.json 2> gpurun_out/bench_ref_r02.err
tail -c 300 gpurun_out/bench_ref_r02.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02.csv \
  python bench.py --steps 2 --warmup 3 --no-moe --no-afd --no-long --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mfa_decode_kernel -s 3 -c 1 -o gpurun_out/r02_mfa_core \
  python bench.py --steps 3 --warmup 3 --workload attn --no-cpu-baseline --no-moe --no-afd --no-long --no-fp8kv > /dev/null 2>&1
ncu -i gpurun_out/r02_mfa_core.ncu-rep --page raw --csv > gpurun_out/r02_mfa_core_raw.csv 2>/dev/null
timeout 600 ncu --set full --clock-control none -k regex:'moe_gemm_mx2_kernel|moe_gemm_bf16_kernel' -c 4 -o gpurun_out/r02_moe \
  python scripts/moe_fmt_bench.py mx:4096 bf16:4096 > /dev/null 2>&1
ncu -i gpurun_out/r02_moe.ncu-rep --page raw --csv > gpurun_out/r02_moe_raw.csv 2>/dev/null
ls -la gpurun_out | tail -12
