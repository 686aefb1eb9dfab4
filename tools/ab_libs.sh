#!/bin/bash
# A/B of library variants (tools/build_variant.sh): e2e phases of a config per variant.
#   VARIANTS="head minb3" CONFIGS="c2 c4" bash tools/ab_libs.sh
for cfg in ${CONFIGS:-c2 c4}; do
  for v in main ${VARIANTS}; do
    lib=paper_2008_03095_b200/lib/variants/libinfuser_b200_$v.so
    [ $v = main ] && lib=paper_2008_03095_b200/lib/libinfuser_b200.so
    echo "== $cfg $v"
    INFUSER_B200_LIB=$PWD/$lib IMX_CELF_PROFILE=1 python tools/e2e_phases.py $cfg 2>&1 | grep -E "^\[celf\]|wall|^device" | tail -${TAIL:-4}
  done
done
