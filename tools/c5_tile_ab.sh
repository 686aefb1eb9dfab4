#!/bin/bash
run() { echo -n "$* : "; env "$@" python tools/ncu_driver.py c5 3 | grep -v src_hash; }
run IMX_TILE_LANES=64 IMX_COMPRESS_WINDOW=32
run IMX_TILE_LANES=128 IMX_COMPRESS_WINDOW=32
run IMX_TILE_LANES=64
run IMX_TILE_LANES=32
