#!/bin/bash
# last check of the final tree (4 GPUs): the whole GPU suite with parity records, smoke, the N=1 bench line
set -u
mkdir -p gpurun_out
export PYTHONPATH=$PWD
PARITY_LOG=gpurun_out/parity_final4.jsonl timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/gputest_final4.log 2>&1
tail -4 gpurun_out/gputest_final4.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/bench_n1_final4.json 2> gpurun_out/bench_n1_final4.err
tail -c 300 gpurun_out/bench_n1_final4.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_n1_final4.json').read().strip().splitlines()[-1])
print('value', round(d['value']), 'e2e', round(d['e2e']['value']), 'us/layer', round(d['ms_per_step']*1e3,1), 'core frac', round(d['roofline']['frac'],3), 'clocks', d['clocks'])"
