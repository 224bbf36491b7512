#!/bin/bash
# round-2 4-GPU session: NVLS + AFD runtime tests across 4 GPUs, NVLS timing, 4-GPU bench with the AFD sweep
set -u
mkdir -p gpurun_out
PARITY_LOG=gpurun_out/parity_r02i.jsonl timeout 1200 python -m pytest tests/test_nvls_gpu.py tests/test_afd_gpu.py \
  tests/test_multi_device_gpu.py -q -rs > gpurun_out/gputest_r02i_4gpu.log 2>&1
tail -3 gpurun_out/gputest_r02i_4gpu.log
for n in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2960$n \
    tests/nvls_check.py --out gpurun_out/nvls_n$n.json > gpurun_out/nvls_n$n.log 2>&1; tail -1 gpurun_out/nvls_n$n.log
done
AFDK_TRACE_DIR=gpurun_out/traces_n4 timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
  --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/bench_n4_r02.json 2> gpurun_out/bench_n4_r02.err
tail -c 600 gpurun_out/bench_n4_r02.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_n4_r02.json").read().strip().splitlines()[-1])
print("value", d["value"], "e2e", d["e2e"]["value"])
for r in d["afd"].get("runs", []):
    if "error" in r:
        print("ERR", r); continue
    print(r["plan"], r["layer"], r["ffn_format"], r["kv"], r["f2a"], r["T_mb"], round(r["layer_period_ms"], 3), round(r["tokens_per_s_per_gpu_per_layer"]), "tpot", round(r["tpot_ms_61_layers"], 1), "sla", r["sla_ok"], "tgs", round(r["tgs_tok_per_gpu_s"]), "stage", {k: round(v) for k, v in r["measured_stage_us"].items()}, r["vet_stages"]["stage_ok"])
print("best_sla", d["afd"].get("best_within_sla"))
PY
