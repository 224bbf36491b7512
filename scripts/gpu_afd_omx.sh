#!/bin/bash
# AFD with MXFP8 o_proj on the attention rank: runtime parity + the 4-GPU AFD lines
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests/test_afd_gpu.py -q -x -k "o-mx or 4r or 2r-1A-mx" 2>&1 | tail -3
for r in 1 2; do
  AFDK_TRACE_DIR=gpurun_out/traces_omx timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 2958$r bench.py --gpus 4 --steps 5 --warmup 3 --no-moe --no-long > gpurun_out/afd_omx_$r.json 2>/dev/null
  python - $r <<'PY'
import json, sys
r = sys.argv[1]
d = json.loads(open(f"gpurun_out/afd_omx_{r}.json").read().strip().splitlines()[-1])
for x in d["afd"].get("runs", []):
    if "error" in x:
        print("ERR", x); continue
    if x["plan"] != "1A3F" or x["kv"] != "e4m3" or x["f2a"] != "nvls":
        continue
    print(x["attn_o_proj"], x["T_mb"], round(x["layer_period_ms"], 3), "tpot", round(x["tpot_ms_61_layers"], 1), "sla", x["sla_ok"], "tgs", round(x["tgs_tok_per_gpu_s"]), {k: round(y) for k, y in x["measured_stage_us"].items()}, x["vet_stages"]["stage_ok"])
b = d["afd"].get("best_within_sla")
print("best", b and (b["attn_o_proj"], b["T_mb"], round(b["tpot_ms_61_layers"], 1), round(b["tgs_tok_per_gpu_s"])))
PY
done
