# A/B of the per-segment work charge (AFDK_MFA_SEG_COST) on the attention core and the config-2 layer
for r in 1 2; do for v in "" _seg0 _seg1 _seg3 _seg4; do
  for cfg in "64 4096" "32 32768" "8 4096"; do
    echo "lib=$v $cfg: $(AFDK_LIB=$PWD/paper_2507_19427_b200/libafdk$v.so timeout 120 python scripts/bench_attn_fp8.py $cfg 2>&1 | tr '\n' '|')"
  done
  echo "lib=$v layer: $(AFDK_LIB=$PWD/paper_2507_19427_b200/libafdk$v.so timeout 120 python scripts/graph_layer.py 2>&1 | tr '\n' ' ')"
done; done
