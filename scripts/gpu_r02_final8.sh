#!/bin/bash
# 4-GPU bench line on the final tree with the AFD sweep extended to T_mb 400 / 416 (bf16 o_proj)
set -u
mkdir -p gpurun_out
export PYTHONPATH=$PWD
: # tests already run on this tree (final6)


timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
AFDK_TRACE_DIR=gpurun_out/traces_final8_n4 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
  --master-addr 127.0.0.1 --master-port 29588 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/bench_final8_n4.json 2> gpurun_out/bench_final8_n4.err
tail -c 200 gpurun_out/bench_final8_n4.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_final8_n4.json").read().strip().splitlines()[-1])
print("N 4 value", round(d["value"]), "e2e", round(d["e2e"]["value"]))
for r in d["afd"].get("runs", []):
    if "error" in r:
        print("ERR", r); continue
    print(r["plan"], r["ffn_format"], r["kv"], r["f2a"], r["attn_o_proj"], r["T_mb"], round(r["layer_period_ms"], 3), "tpot", round(r["tpot_ms_61_layers"], 1), "sla", r["sla_ok"], "tgs", round(r["tgs_tok_per_gpu_s"]), {k: round(v) for k, v in r["measured_stage_us"].items()})
b = d["afd"].get("best_within_sla")
print("best_sla", b and (b["plan"], b["attn_o_proj"], b["T_mb"], round(b["tpot_ms_61_layers"], 1), round(b["tgs_tok_per_gpu_s"])))
PY
