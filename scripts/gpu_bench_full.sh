# the driver's scaling command shape: bash scripts/gpu_bench_full.sh N
N=${1:-2}
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus $N > gpurun_out/full$N.json 2> gpurun_out/full$N.err
echo "rc=$?"; tail -c 300 gpurun_out/full$N.err
