#!/bin/bash
# AFD FFN direct mode (in-place payload, flag wait in the permute kernel): parity + A/B (4 GPUs)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 1500 python -m pytest tests/test_afd_gpu.py tests/test_afd_cpp_gpu.py -q -x -k "not 8r" 2>&1 | tail -3
for v in 1 0 1 0; do
  AFDK_AFD_DIRECT=$v timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 2957$v bench.py --gpus 4 --steps 5 --warmup 3 --no-moe --no-long > gpurun_out/ab_direct_$v.json 2>/dev/null
  python - $v <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads(open(f"gpurun_out/ab_direct_{v}.json").read().strip().splitlines()[-1])
for x in d["afd"].get("runs", []):
    if "error" in x:
        print("ERR", x); continue
    if x["plan"] != "1A3F" or x["kv"] != "e4m3":
        continue
    print("direct", v, x["ffn_format"], x["f2a"], x["T_mb"], round(x["layer_period_ms"], 3), "tpot", round(x["tpot_ms_61_layers"], 1), "tgs", round(x["tgs_tok_per_gpu_s"]), {k: round(y) for k, y in x["measured_stage_us"].items()}, x["vet_stages"]["stage_ok"])
PY
done
