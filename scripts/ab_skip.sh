for r in 1 2; do
for m in 0 1 2 4 8 16 32 64 128 5 6 24 96 160 255; do
  echo "skip=$m $(AFDK_LAYER_SKIP=$m timeout 120 python scripts/graph_layer.py 2>&1 | tr '\n' ' ')"
done
done
