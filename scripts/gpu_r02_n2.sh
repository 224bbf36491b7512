#!/bin/bash
# round-2 2-GPU session: NVLS + AFD runtime (cross-GPU) tests, MX SiLU A/B, 2-GPU bench with the AFD sweep
set -u
mkdir -p gpurun_out
PARITY_LOG=gpurun_out/parity_r02h.jsonl timeout 1200 python -m pytest tests/test_nvls_gpu.py tests/test_afd_gpu.py \
  tests/test_multi_device_gpu.py -q -rs > gpurun_out/gputest_r02h_2gpu.log 2>&1
tail -3 gpurun_out/gputest_r02h_2gpu.log
for i in 1 2; do
  CUDA_VISIBLE_DEVICES=0 AFDK_LIB=paper_2507_19427_b200/libafdk_silexp.so timeout 300 python scripts/moe_fmt_bench.py mx:4096 mx:8192 bf16:4096 2>/dev/null | cut -c1-90 | sed 's/^/exp  /'
  CUDA_VISIBLE_DEVICES=0 timeout 300 python scripts/moe_fmt_bench.py mx:4096 mx:8192 bf16:4096 2>/dev/null | cut -c1-90 | sed 's/^/tanh /'
done
AFDK_TRACE_DIR=gpurun_out/traces_n2 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_n2_r02.json 2> gpurun_out/bench_n2_r02.err
tail -c 600 gpurun_out/bench_n2_r02.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_n2_r02.json").read().strip().splitlines()[-1])
print("value", d["value"], "e2e", d["e2e"]["value"])
for r in d["afd"].get("runs", []):
    print(r["plan"], r["layer"], r["ffn_format"], r["kv"], r["T_mb"], round(r["layer_period_ms"], 3), round(r["tokens_per_s_per_gpu_per_layer"]), "tpot", round(r["tpot_ms_61_layers"], 1), "sla", r["sla_ok"], "tgs", round(r["tgs_tok_per_gpu_s"]), "stage", {k: round(v) for k, v in r["measured_stage_us"].items()}, r["vet_stages"]["stage_ok"])
print("best_sla", d["afd"].get("best_within_sla"))
PY
