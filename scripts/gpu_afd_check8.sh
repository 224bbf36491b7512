# The 8-rank AFD protocol (2A6F, 4A4F) on a 4-GPU box: two ranks per GPU, gloo rendezvous, --check only
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29519"
export AFDK_OVERSUB=1
timeout 300 $T scripts/afd_run.py --n-attn 2 --check --fmt mx --attn-chunk 10 2>&1 | grep -E "afd_check|Error|error" | head -5
timeout 300 $T scripts/afd_run.py --n-attn 2 --check --fmt fp8 --f2a pull 2>&1 | grep -E "afd_check|Error|error" | head -5
timeout 300 $T scripts/afd_run.py --n-attn 4 --check --fmt mx 2>&1 | grep -E "afd_check|Error|error" | head -5
timeout 300 $T scripts/afd_run.py --n-attn 4 --check --fmt mx --layer dense 2>&1 | grep -E "afd_check|Error|error" | head -5
