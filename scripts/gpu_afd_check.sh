# AFD correctness (moe/dense, push/pull, fp8/mx, chunked attention): bash scripts/gpu_afd_check.sh N
N=${1:-2}
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513"
timeout 180 $T scripts/afd_run.py --n-attn 1 --check --fmt mx --attn-chunk 10 2>&1 | grep afd_check
timeout 180 $T scripts/afd_run.py --n-attn 1 --check --fmt fp8 --f2a pull --attn-chunk 7 2>&1 | grep afd_check
timeout 180 $T scripts/afd_run.py --n-attn 1 --check --fmt mx --layer dense 2>&1 | grep afd_check
