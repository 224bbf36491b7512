# A/B of the MXFP8 MoE layer between the current library and libafdk_old256.so
for r in 1 2; do for v in "" _old256; do
  for T in 1024 2048 4096 5120 8192; do
    echo "lib=$v T=$T: $(AFDK_LIB=$PWD/paper_2507_19427_b200/libafdk$v.so timeout 120 python scripts/prof_moe.py $T mx 2>&1 | tail -1)"
  done
done
echo "chunk256 T=4096: $(AFDK_MX_CHUNK=256 timeout 120 python scripts/prof_moe.py 4096 mx 2>&1 | tail -1)"
done
