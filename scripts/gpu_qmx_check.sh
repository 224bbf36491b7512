#!/bin/bash
# AFD runtime with MXFP8 q_up + o_proj on the attention rank: small dims (2 ranks) and Step-3 dims (4 ranks)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 600 python -m pytest tests/test_afd_gpu.py -q -x -k "e4m3-2" 2>&1 | tail -15
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 \
  tests/afd_gpu_check.py --n-attn 1 --fmt mx --f2a nvls --kv e4m3 --T-mb 368 --attn-chunk 512 --steps 2 --layers 1 --full 1 --o-mx 2 \
  --out gpurun_out/qmx_full.json 2>&1 | tail -8
cat gpurun_out/qmx_full.json 2>/dev/null | head -c 600
