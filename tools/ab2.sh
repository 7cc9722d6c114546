#!/bin/bash
# A/B of libinim builds on one box (run under gpurun): C2 and C3 graph-replay slopes and
# the integral sweep, interleaved, each build twice.   bash tools/ab2.sh ab/libA.so ab/libB.so ...
sw() { tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(' '.join('%d:%.0f' % (r['size'], r['GB_s']) for r in d['sweep']))"; }
for rep in 1 2; do
  for L in "$@"; do
    echo "$L c2 $(INIM_LIB_PATH=$L python tools/run_probe.py | tail -1)"
  done
done
for L in "$@"; do
  echo "$L c3 $(INIM_LIB_PATH=$L python tools/run_probe.py c3 | tail -1)"
  echo "$L sweep $(INIM_LIB_PATH=$L python bench.py --workload sweep --steps 10 2>/dev/null | sw)"
done
