# A/B of the config-2 layer between the current library and libafdk_prev.so
for r in 1 2 3; do for v in "" _prev; do
  echo "lib=$v $(AFDK_LIB=$PWD/paper_2507_19427_b200/libafdk$v.so timeout 120 python scripts/graph_layer.py 2>&1 | tr '\n' ' ')"
done; done
