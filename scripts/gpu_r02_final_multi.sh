#!/bin/bash
# final round-2 multi-GPU session: 2/4-GPU tests, 2- and 4-GPU bench lines with AFD traces
set -u
mkdir -p gpurun_out
PARITY_LOG=gpurun_out/parity_final_multi.jsonl timeout 1200 python -m pytest tests/test_nvls_gpu.py tests/test_afd_gpu.py \
  tests/test_multi_device_gpu.py -q -rs > gpurun_out/gputest_final_multi.log 2>&1
tail -3 gpurun_out/gputest_final_multi.log
for n in 4 2; do
  AFDK_TRACE_DIR=gpurun_out/traces_final_n$n timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port 2952$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/bench_final_n$n.json 2> gpurun_out/bench_final_n$n.err
  tail -c 300 gpurun_out/bench_final_n$n.err
  python - $n <<'PY'
import json, sys
n = sys.argv[1]
d = json.loads(open(f"gpurun_out/bench_final_n{n}.json").read().strip().splitlines()[-1])
print("N", n, "value", round(d["value"]), "e2e", round(d["e2e"]["value"]))
for r in d["afd"].get("runs", []):
    if "error" in r:
        print("ERR", r); continue
    print(r["plan"], r["layer"], r["ffn_format"], r["kv"], r["f2a"], r["T_mb"], round(r["layer_period_ms"], 3), round(r["tokens_per_s_per_gpu_per_layer"]), "tpot", round(r["tpot_ms_61_layers"], 1), "sla", r["sla_ok"], "tgs", round(r["tgs_tok_per_gpu_s"]), {k: round(v) for k, v in r["measured_stage_us"].items()}, r["vet_stages"]["stage_ok"])
b = d["afd"].get("best_within_sla")
print("best_sla", b and (b["plan"], b["ffn_format"], b["kv"], b["f2a"], b["T_mb"], round(b["tpot_ms_61_layers"], 1), round(b["tgs_tok_per_gpu_s"])))
PY
done
