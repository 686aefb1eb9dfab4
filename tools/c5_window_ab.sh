#!/bin/bash
# C5 compress: tiled copies (default) vs in-place lane windows, with and without row-stride padding
run() { echo -n "$* : "; env "$@" python tools/ncu_driver.py c5 3 | grep -v src_hash; }
run IMX_COMPRESS_TILE=32
for pad in 0 32 96; do
  for win in 32 64 128; do
    run IMX_LD_PAD=$pad IMX_COMPRESS_TILE=0 IMX_COMPRESS_WINDOW=$win
  done
done
run IMX_LD_PAD=32 IMX_COMPRESS_TILE=0
