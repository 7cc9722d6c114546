#!/bin/bash
# Tile geometry vs the C2 iteration (run on the GPU box):
#   bash tools/geo_sweep_c2.sh > gpurun_out/geo_sweep_c2.txt
for th in 4 8 16; do
  for tw in 32 64 128; do
    r=$(INIM_GEO_TH=$th INIM_GEO_TW=$tw timeout 300 python bench.py --no-cpu-baseline --steps 10 2>&1 | tail -1 |
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.0f iters/s' % d['value'], ' '.join('%s:%.1f' % (k, v['avg_us']) for k, v in d['kernels'].items()))" 2>&1 | tail -1)
    echo "TH=$th TW=$tw  $r"
  done
done
