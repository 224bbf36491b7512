# A/B of the MXFP8 MoE layer (and dense FFN) between the current library and libafdk_v2.so
for r in 1 2; do for v in "" _v2; do
  for T in 512 1024 2048 3072 4096 8192; do
    echo "lib=$v T=$T: $(AFDK_LIB=$PWD/paper_2507_19427_b200/libafdk$v.so timeout 120 python scripts/prof_moe.py $T mx 2>&1 | tail -1)"
  done
  echo "lib=$v dense: $(AFDK_LIB=$PWD/paper_2507_19427_b200/libafdk$v.so timeout 120 python scripts/prof_dense.py 4096 4 2>&1 | tail -1)"
done; done
