#!/bin/bash
# A/B of libinim builds on the SPLOM batch (run under gpurun): bash tools/ab_splom.sh ab/libA.so ab/libB.so ...
for rep in 1 2; do
  for L in "$@"; do
    echo "$L $(INIM_LIB_PATH=$L python tools/splom_probe.py 256 256 | tail -1)"
  done
done
