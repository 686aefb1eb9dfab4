#!/bin/bash
# Build a variant of libinfuser_b200.so with extra nvcc defines, for A/B runs:
#   tools/build_variant.sh TAG -DNAME=VALUE ...  ->  paper_2008_03095_b200/lib/variants/libinfuser_b200_TAG.so
# select it with INFUSER_B200_LIB=<path>.  CSRC=<dir> compiles another copy of
# the sources (e.g. a git worktree's csrc) instead of the tree's.
set -e
cd "$(dirname "$0")/.."
tag=$1; shift
src=${CSRC:-paper_2008_03095_b200/csrc}
out=paper_2008_03095_b200/lib/variants/$tag
mkdir -p $out
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -diag-suppress 1444 -Iinclude $*"
objs=""
for s in graph.cu gen.cu ctx.cu propagate.cu scan.cu memo.cu celf.cu comm.cu evaluation.cu upload.cu io.cpp; do
  nvcc $F -c -o $out/$s.o $src/$s 2>/dev/null &
  objs="$objs $out/$s.o"
done
wait
nvcc $F -shared -cudart static -ldl -o paper_2008_03095_b200/lib/variants/libinfuser_b200_$tag.so $objs
echo paper_2008_03095_b200/lib/variants/libinfuser_b200_$tag.so
