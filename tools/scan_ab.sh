#!/bin/bash
# A/B of the sampler strategies: propagate phase times per config
for c in ${CONFIGS:-c4 c5 c2 c2p1 c1}; do
  for m in ${MODES:-scan enum pull}; do
    echo -n "$m "; IMX_HOOK=$m python tools/ncu_driver.py $c 5 | grep -v src_hash
  done
done
