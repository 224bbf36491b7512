#!/bin/bash
# determinism + AFD soak, C++ AFD driver tests, MFA launch timeline (4 GPUs)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 600 python scripts/soak_determinism.py 200 > gpurun_out/soak_det.log 2>&1; echo "det rc=$?"
tail -12 gpurun_out/soak_det.log
for c in "bf16 nvls" "bf16 push" "mx nvls" "bf16 pull"; do
  set -- $c
  for i in 1 2 3; do
    timeout 300 torchrun --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 2960$i tests/afd_gpu_check.py \
      --n-attn 1 --fmt $1 --f2a $2 --steps 12 --out gpurun_out/soak_$1_$2_$i.json > gpurun_out/soak_$1_$2_$i.log 2>&1
    echo "afd $1 $2 run $i rc=$? $(python -c "import json;d=json.load(open('gpurun_out/soak_$1_$2_$i.json'));print(d['afd_check'], round(d['max_rel_err'],4), [round(e,3) for e in d['rel_err'] if e>0.015])" 2>/dev/null)"
  done
done
timeout 900 python -m pytest tests/test_afd_cpp_gpu.py -q -x 2>&1 | tail -5
for a in "64 4096" "64 4096 fp8" "32 32768" "32 32768 fp8" "256 4096 fp8"; do
  AFDK_LIB=$PWD/paper_2507_19427_b200/libafdk_times.so timeout 120 python scripts/mfa_timeline.py $a 2>&1 | tail -9
done
