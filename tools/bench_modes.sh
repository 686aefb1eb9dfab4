#!/bin/bash
# propagate time per sampler strategy and config (tools/ncu_driver.py prints bench_propagate)
for cfg in ${CONFIGS:-c1 c2 c2p1 c3 c5 c4}; do
  for mode in enum pull hybrid; do
    echo -n "$cfg $mode "; IMX_HOOK=$mode timeout 600 python tools/ncu_driver.py $cfg 5 2>&1 | tail -1
  done
done
