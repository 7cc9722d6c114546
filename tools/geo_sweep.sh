#!/bin/bash
# Tile-geometry experiment for the integral pass (run on the GPU box):
#   bash tools/geo_sweep.sh > gpurun_out/geo_sweep.txt
# One process per INIM_GEO_TH/TW pair (the override is read once per process).
for th in 16 32 64; do
  for tw in 64 128; do
    r=$(INIM_GEO_TH=$th INIM_GEO_TW=$tw timeout 300 python bench.py --workload sweep --steps 10 2>/dev/null | tail -1 |
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print(' '.join('%d:%.0f' % (r['size'], r['GB_s']) for r in d['sweep']))")
    echo "TH=$th TW=$tw  $r"
  done
done
