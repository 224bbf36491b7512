#!/bin/bash
# full-dims AFD parity (4 GPUs) + in-kernel-wait REDUCE: parity and A/B
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571 \
  tests/afd_gpu_check.py --n-attn 1 --fmt mx --f2a nvls --kv e4m3 --T-mb 320 --steps 2 --layers 1 --full 1 \
  --out gpurun_out/full_afd.json > gpurun_out/full_afd.log 2>&1; echo "full rc=$?"; tail -c 1500 gpurun_out/full_afd.log
AFDK_AFD_FUSED_WAIT=1 timeout 900 python -m pytest tests/test_afd_gpu.py -q -x -k "not 8r and not 4r" 2>&1 | tail -2
for v in 1 0 1 0; do
  AFDK_AFD_FUSED_WAIT=$v timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 2956$v bench.py --gpus 4 --steps 5 --warmup 3 --no-moe --no-long > gpurun_out/ab_fw_$v.json 2>/dev/null
  python - $v <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads(open(f"gpurun_out/ab_fw_{v}.json").read().strip().splitlines()[-1])
for x in d["afd"].get("runs", []):
    if "error" in x or x["plan"] != "1A3F" or x["kv"] != "e4m3":
        continue
    print("fw", v, x["ffn_format"], x["f2a"], x["T_mb"], round(x["layer_period_ms"], 3), "tpot", round(x["tpot_ms_61_layers"], 1), "tgs", round(x["tgs_tok_per_gpu_s"]), {k: round(y) for k, y in x["measured_stage_us"].items()})
PY
done
