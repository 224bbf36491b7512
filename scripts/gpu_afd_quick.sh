#!/bin/bash
# AFD runs only (4 GPUs), short: the AFD lines of bench.py
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_afd_gpu.py tests/test_afd_cpp_gpu.py -q -x -k "not 8r" 2>&1 | tail -2
for r in 1 2; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 2955$r bench.py --gpus 4 --steps 5 --warmup 3 --no-moe --no-long > gpurun_out/afd_quick_$r.json 2>/dev/null
  python - $r <<'PY'
import json, sys
r = sys.argv[1]
d = json.loads(open(f"gpurun_out/afd_quick_{r}.json").read().strip().splitlines()[-1])
for x in d["afd"].get("runs", []):
    if "error" in x or x["plan"] != "1A3F":
        continue
    print(x["plan"], x["ffn_format"], x["kv"], x["f2a"], x["T_mb"], round(x["layer_period_ms"], 3), "tpot", round(x["tpot_ms_61_layers"], 1), "tgs", round(x["tgs_tok_per_gpu_s"]), {k: round(v) for k, v in x["measured_stage_us"].items()}, x["vet_stages"]["stage_ok"])
PY
done
