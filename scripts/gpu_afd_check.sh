# AFD correctness (push/pull x fp8/mx) and push-vs-pull timing: bash scripts/gpu_afd_check.sh N
N=${1:-2}
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513"
for f2a in push pull; do for fmt in fp8 mx; do
  timeout 180 $T scripts/afd_run.py --n-attn 1 --check --fmt $fmt --f2a $f2a 2>&1 | grep afd_check
done; done
for f2a in push pull; do
  timeout 240 $T scripts/afd_run.py --n-attn $((N / 2)) --T-mb 256 --fmt mx --f2a $f2a --steps 8 2>&1 | grep '"afd"'
done
