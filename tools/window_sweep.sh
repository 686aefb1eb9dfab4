#!/bin/bash
# compress lane-window sweep: propagate time per config and IMX_COMPRESS_WINDOW
for cfg in ${CONFIGS:-c5 c4 c3 c2}; do
  for w in ${WINDOWS:-0 16 32 64 128}; do
    echo -n "$cfg win=$w "; IMX_COMPRESS_WINDOW=$w timeout 600 python tools/ncu_driver.py $cfg 3 2>&1 | tail -1
  done
done
