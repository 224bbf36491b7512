#!/bin/bash
# fused decode MoE kernel: parity, determinism, A/B; AFD soak with per-layer checks (4 GPUs)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_moe_mx_gpu.py tests/test_bench_shapes_gpu.py tests/test_error_budget_gpu.py tests/test_moe_gpu.py -q -x 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python scripts/soak_determinism.py 100 2>&1 | grep mx
bash scripts/ab_fused.sh 2>&1
for c in "bf16 nvls" "bf16 push" "bf16 pull" "mx push" "fp8 pull"; do
  set -- $c
  for i in 1 2; do
    timeout 300 torchrun --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 2961$i tests/afd_gpu_check.py \
      --n-attn 1 --fmt $1 --f2a $2 --steps 12 --out gpurun_out/soak2_$1_$2_$i.json > gpurun_out/soak2_$1_$2_$i.log 2>&1
    echo "afd $1 $2 run $i rc=$? $(python -c "import json;d=json.load(open('gpurun_out/soak2_$1_$2_$i.json'));print(d['afd_check'], round(d['max_rel_err'],4), len(d['rel_err']))" 2>/dev/null)"
  done
done
timeout 900 python -m pytest tests/test_afd_cpp_gpu.py tests/test_afd_gpu.py -q 2>&1 | tail -4
