# AFD bench sweep on N GPUs of one box: bash scripts/gpu_afd.sh N  (run under gpurun --gpus N)
set -o pipefail
N=${1:-2}
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511"
timeout 480 $T bench.py --gpus $N --steps 8 --warmup 3 --no-moe --no-long --no-fp8kv > gpurun_out/afd$N.json 2> gpurun_out/afd$N.err
tail -3 gpurun_out/afd$N.err
