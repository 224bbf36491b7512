# MXFP8 MoE: parity (both kernels), layer timings, MMA-issuer wait profile
timeout 300 python -m pytest tests/test_moe_mx_gpu.py -x -q 2>&1 | tail -2
for T in 256 1024 4096 8192; do timeout 120 python scripts/prof_moe.py $T mx; done
if [ -f paper_2507_19427_b200/libafdk_prof.so ]; then
  AFDK_LIB=paper_2507_19427_b200/libafdk_prof.so timeout 120 python scripts/prof_moe.py 8192 mx 2>&1 | grep "pair 0 " | tail -2
fi
