#!/bin/bash
# MXFP8 q_up on the attention side: parity (layer + AFD runtime), layer A/B, 4-GPU AFD lines
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_mfa_layer_gpu.py tests/test_linear_mx_gpu.py -q -x -k "mx" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_afd_gpu.py -q -x -k "e4m3-1 or e4m3-2" 2>&1 | tail -2
for b in 64 352; do
  timeout 600 python bench.py --steps 10 --warmup 3 --batch $b --no-moe --no-afd --no-long --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); f=d['config2_fp8_kv']; m=f['layer_mx_oproj']
print('B=$b bf16 layer', round(d['ms_per_step']*1e3,1), 'e4m3 layer', round(f['layer_ms']*1e3,1), 'o_mx', round(m['layer_ms']*1e3,1), 'o+q_up mx', round(m['with_q_up_mx']['layer_ms']*1e3,1))"
done
for r in 1 2; do
  AFDK_TRACE_DIR=gpurun_out/traces_qmx timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 2959$r bench.py --gpus 4 --steps 5 --warmup 3 --no-moe --no-long > gpurun_out/afd_qmx_$r.json 2>/dev/null
  python - $r <<'PY'
import json, sys
r = sys.argv[1]
d = json.loads(open(f"gpurun_out/afd_qmx_{r}.json").read().strip().splitlines()[-1])
for x in d["afd"].get("runs", []):
    if "error" in x:
        print("ERR", x); continue
    if x["plan"] != "1A3F" or x["kv"] != "e4m3" or x["f2a"] != "nvls":
        continue
    print(x["attn_o_proj"], x.get("attn_q_up"), x["T_mb"], round(x["layer_period_ms"], 3), "tpot", round(x["tpot_ms_61_layers"], 1), "sla", x["sla_ok"], "tgs", round(x["tgs_tok_per_gpu_s"]), {k: round(y) for k, y in x["measured_stage_us"].items()}, x["vet_stages"]["stage_ok"])
b = d["afd"].get("best_within_sla")
print("best", b and (b["attn_o_proj"], b.get("attn_q_up"), b["T_mb"], round(b["tpot_ms_61_layers"], 1), round(b["tgs_tok_per_gpu_s"])))
PY
done
