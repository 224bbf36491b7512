#!/bin/bash
# router top-k epilogue with coalesced partial loads: parity (router, MoE, AFD runtime incl. C++), launch list, 4-GPU bench line
set -u
mkdir -p gpurun_out
export PYTHONPATH=$PWD
PARITY_LOG=gpurun_out/parity_final9.jsonl timeout 1800 python -m pytest tests/test_moe_gpu.py tests/test_moe_mx_gpu.py tests/test_moe_bf16_gpu.py \
  tests/test_bench_shapes_gpu.py tests/test_error_budget_gpu.py tests/test_afd_gpu.py tests/test_afd_cpp_gpu.py tests/test_stage_times_gpu.py -q -x > gpurun_out/gputest_final9.log 2>&1
tail -2 gpurun_out/gputest_final9.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/afd_attn_launches9.csv python scripts/prof_afd_attn.py 384 1 > /dev/null 2>&1
AFDK_TRACE_DIR=gpurun_out/traces_final9_n4 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
  --master-addr 127.0.0.1 --master-port 29589 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/bench_final9_n4.json 2> gpurun_out/bench_final9_n4.err
tail -c 200 gpurun_out/bench_final9_n4.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_final9_n4.json").read().strip().splitlines()[-1])
print("N 4 value", round(d["value"]), "e2e", round(d["e2e"]["value"]))
for r in d["afd"].get("runs", []):
    if "error" in r:
        print("ERR", r); continue
    if r["plan"] == "1A3F" and r["f2a"] == "nvls":
        print(r["attn_o_proj"], r["T_mb"], round(r["layer_period_ms"], 3), "tpot", round(r["tpot_ms_61_layers"], 1), "sla", r["sla_ok"], "tgs", round(r["tgs_tok_per_gpu_s"]), {k: round(v) for k, v in r["measured_stage_us"].items()})
b = d["afd"].get("best_within_sla")
print("best_sla", b and (b["plan"], b["attn_o_proj"], b["T_mb"], round(b["tpot_ms_61_layers"], 1), round(b["tgs_tok_per_gpu_s"])))
PY
