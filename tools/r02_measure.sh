#!/bin/bash
# ncu per-config summaries at this source hash, then the bench arms.
#   CONFIGS="c4 c5" BENCH="c4" bash tools/r02_measure.sh
set -x
mkdir -p gpurun_out
CONFIGS="${CONFIGS:-c4}" bash tools/ncu_configs.sh
for cfg in ${CONFIGS:-c4}; do
  python tools/ncu_summarize.py $cfg gpurun_out/ncu_$cfg.csv > gpurun_out/ncu_sum_$cfg.txt 2>&1
  cp profiles/ncu_${cfg}_summary.json gpurun_out/ 2>/dev/null
done
for cfg in ${BENCH:-c4}; do
  python bench.py --config $cfg ${BENCH_ARGS} > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
  [ -n "$REF" ] && python bench.py --config $cfg --impl reference > gpurun_out/ref_$cfg.json 2> gpurun_out/ref_$cfg.err
done
true
