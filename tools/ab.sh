#!/bin/bash
# A/B timing of two builds of libinim.so on the same box (run under gpurun):
#   bash tools/ab.sh abtest/libinim_base.so [extra env for B...]
# A = the given build, B = the in-tree build; each measured twice, interleaved.
A=$1; shift
sw() { tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(' '.join('%d:%.0f' % (r['size'], r['GB_s']) for r in d['sweep']))"; }
for rep in 1 2; do
  echo "A c2  $(INIM_LIB_PATH=$A python tools/run_probe.py | tail -1)"
  echo "B c2  $(env "$@" python tools/run_probe.py | tail -1)"
  echo "A c3  $(INIM_LIB_PATH=$A python tools/run_probe.py c3 | tail -1)"
  echo "B c3  $(env "$@" python tools/run_probe.py c3 | tail -1)"
  echo "A sweep $(INIM_LIB_PATH=$A python bench.py --workload sweep --steps 10 2>/dev/null | sw)"
  echo "B sweep $(env "$@" python bench.py --workload sweep --steps 10 2>/dev/null | sw)"
done
