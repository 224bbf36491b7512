# A/B of the current library against libafdk_oldk3.so: attention core (bf16 / e4m3 / mtp) and the config-2 layer
for r in 1 2; do for v in "" _oldk3; do
  for cfg in "64 4096" "32 32768" "8 4096"; do
    echo "lib=$v $cfg: $(AFDK_LIB=$PWD/paper_2507_19427_b200/libafdk$v.so timeout 120 python scripts/bench_attn_fp8.py $cfg 2>&1 | tr '\n' '|')"
  done
  echo "lib=$v layer: $(AFDK_LIB=$PWD/paper_2507_19427_b200/libafdk$v.so timeout 120 python scripts/graph_layer.py 2>&1 | tr '\n' ' ')"
done; done
