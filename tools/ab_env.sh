#!/bin/bash
# A/B of one build under environment settings (run under gpurun), interleaved, twice:
#   bash tools/ab_env.sh "INIM_X=0" "INIM_X=1" ...      (SPLOM batch, C2 and C3 probes)
for rep in 1 2; do
  for E in "$@"; do
    echo "$E splom $(env $E python tools/splom_probe.py 256 256 | tail -1)"
    echo "$E c2 $(env $E python tools/run_probe.py | tail -1)"
  done
done
for E in "$@"; do
  echo "$E c3 $(env $E python tools/run_probe.py c3 | tail -1)"
done
