#!/bin/bash
# Run bench.py on every BASELINE config (1 GPU); one JSON line per config.
mkdir -p gpurun_out
for cfg in ${CONFIGS:-c1 c2 c2p1 c3 c5 c4}; do
  extra=""
  case $cfg in c4|c5) extra="--e2e-steps 1 --cpu-budget-s 10";; esac
  timeout 900 python bench.py --config $cfg --steps ${STEPS:-5} --warmup 3 $extra \
      > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
  echo "$cfg rc=$?"
done
