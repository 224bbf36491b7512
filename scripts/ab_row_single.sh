#!/bin/bash
# row epilogues (input RMSNorm, o epilogue) with one CTA per row from 128 rows: parity + A/B (1 GPU)
cd "$(dirname "$0")/.."
export PYTHONPATH=$PWD
export AFDK_LIB=$PWD/paper_2507_19427_b200/libafdk_rowsingle.so
AFDK_ROW_SINGLE=1 timeout 900 python -m pytest tests/test_mfa_layer_gpu.py -q -x 2>&1 | tail -2
for r in 1 2; do
  for v in 1 0; do
    for B in 128 256 320 384; do
      echo "single=$v B=$B: $(AFDK_ROW_SINGLE=$v timeout 600 python bench.py --steps 10 --warmup 3 --batch $B --no-moe --no-afd --no-long --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step']*1e3,1), 'us/layer bf16; e4m3', round(d['config2_fp8_kv']['layer_ms']*1e3,1))")"
    done
  done
done
