#!/bin/bash
# A/B: AFD attention ranks with serialised attention compute (AFDK_AFD_ATTN_SERIAL) (4 GPUs)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONPATH=$PWD
AFDK_AFD_ATTN_SERIAL=1 timeout 900 python -m pytest tests/test_afd_gpu.py -q -x -k "not 8r" 2>&1 | tail -2
for v in 1 0 1 0; do
  AFDK_AFD_ATTN_SERIAL=$v timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 2954$v bench.py --gpus 4 --steps 5 --warmup 3 --no-moe --no-long > gpurun_out/ab_serial_$v.json 2>/dev/null
  python - $v <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads(open(f"gpurun_out/ab_serial_{v}.json").read().strip().splitlines()[-1])
for r in d["afd"].get("runs", []):
    if "error" in r or r["plan"] != "1A3F":
        continue
    print("serial", v, r["plan"], r["ffn_format"], r["kv"], r["f2a"], r["T_mb"], round(r["layer_period_ms"], 3), "tpot", round(r["tpot_ms_61_layers"], 1), "tgs", round(r["tgs_tok_per_gpu_s"]), {k: round(x) for k, x in r["measured_stage_us"].items()}, r["vet_stages"]["stage_ok"])
PY
done
