for r in 1 2 3; do
  echo "stream-K $(AFDK_LIB=$PWD/paper_2507_19427_b200/libafdk_tg.so timeout 120 python scripts/graph_layer.py 2>&1 | tr '\n' ' ')"
  echo "tile-grid $(AFDK_TILE_GRID=1 AFDK_LIB=$PWD/paper_2507_19427_b200/libafdk_tg.so timeout 120 python scripts/graph_layer.py 2>&1 | tr '\n' ' ')"
done
