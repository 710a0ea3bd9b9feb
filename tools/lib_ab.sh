#!/bin/bash
# Interleaved A/B of whole config-3 refinements between libsr builds, one
# process per measurement, alternating: bash tools/lib_ab.sh ROUNDS libA.so libB.so ...
# ("main" = the in-tree build)
rounds=$1; shift
for r in $(seq 1 $rounds); do
  for lib in "$@"; do
    if [ "$lib" = main ]; then L=""; else L=$lib; fi
    echo "$lib $(SR_LIB_PATH=$L python tools/time_config3.py 3 2>/dev/null | tail -1)"
  done
done
