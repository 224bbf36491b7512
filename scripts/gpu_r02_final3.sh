#!/bin/bash
# round-2 third final session (4 GPUs): the whole GPU suite, N=1 bench + launch list,
# ncu of the fused decode MoE kernel, 4- and 2-GPU bench lines with AFD traces
set -u
mkdir -p gpurun_out
export PYTHONPATH=$PWD
PARITY_LOG=gpurun_out/parity_final3.jsonl timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/gputest_final3.log 2>&1
tail -4 gpurun_out/gputest_final3.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/bench_n1_final3.json 2> gpurun_out/bench_n1_final3.err
tail -c 300 gpurun_out/bench_n1_final3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final3.csv \
  python bench.py --steps 2 --warmup 3 --no-moe --no-afd --no-long --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:moe_ffn_mx_fused_kernel -s 2 -c 1 -o gpurun_out/r02_fused \
  python scripts/prof_moe_shard.py 256 3 mx > /dev/null 2>&1
ncu -i gpurun_out/r02_fused.ncu-rep --page raw --csv > gpurun_out/r02_fused_raw.csv 2>/dev/null
for n in 4 2; do
  AFDK_TRACE_DIR=gpurun_out/traces_final3_n$n timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/bench_final3_n$n.json 2> gpurun_out/bench_final3_n$n.err
  tail -c 300 gpurun_out/bench_final3_n$n.err
  python - $n <<'PY'
import json, sys
n = sys.argv[1]
d = json.loads(open(f"gpurun_out/bench_final3_n{n}.json").read().strip().splitlines()[-1])
print("N", n, "value", round(d["value"]), "e2e", round(d["e2e"]["value"]))
for r in d["afd"].get("runs", []):
    if "error" in r:
        print("ERR", r); continue
    print(r["plan"], r["layer"], r["ffn_format"], r["kv"], r["f2a"], r["T_mb"], round(r["layer_period_ms"], 3), round(r["tokens_per_s_per_gpu_per_layer"]), "tpot", round(r["tpot_ms_61_layers"], 1), "sla", r["sla_ok"], "tgs", round(r["tgs_tok_per_gpu_s"]), {k: round(v) for k, v in r["measured_stage_us"].items()}, r["vet_stages"]["stage_ok"])
b = d["afd"].get("best_within_sla")
print("best_sla", b and (b["plan"], b["ffn_format"], b["kv"], b["f2a"], b["T_mb"], round(b["tpot_ms_61_layers"], 1), round(b["tgs_tok_per_gpu_s"])))
PY
done
