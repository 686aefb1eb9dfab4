#!/bin/bash
# End-of-round measurement: ncu per-config summaries at this source hash, bench lines of
# every config (ours + reference arm), launch lists, one --set full capture of the two
# longest C4 kernels.  Everything lands in gpurun_out/final/.
set -x
O=gpurun_out/final
mkdir -p $O
CFGS="${CONFIGS:-c1 c2 c2p1 c3 c4 c5}"
# 1. per-config ncu summaries (stamps profiles/ncu_<cfg>_summary.json with the source hash)
CONFIGS="$CFGS" bash tools/ncu_configs.sh
for cfg in $CFGS; do
  python tools/ncu_summarize.py $cfg gpurun_out/ncu_$cfg.csv > $O/ncu_$cfg.txt 2>&1
  cp profiles/ncu_${cfg}_summary.json $O/ 2>/dev/null
done
# 2. bench lines
for cfg in $CFGS; do
  extra=""
  case $cfg in c5) extra="--e2e-steps 3";; esac
  timeout 1200 python bench.py --config $cfg $extra > $O/bench_$cfg.json 2> $O/bench_$cfg.err
  echo "bench $cfg rc=$?"
  timeout 900 python bench.py --config $cfg --impl reference --steps 3 --warmup 1 > $O/ref_$cfg.json 2> $O/ref_$cfg.err
  echo "ref $cfg rc=$?"
done
# 3. launch list of the default bench command (cold-cache, serialised: shares only)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_c4_bench.csv \
    python bench.py --steps 2 --warmup 1 --parity off --no-cpu-baseline --e2e-steps 1 > $O/launches_c4_bench.log 2>&1
echo "launch list rc=$?"
# 4. --set full of the two longest C4 kernels (R = 256 lanes so that kernel replay can save the matrix);
#    ncu matches the function name without template arguments: k_scan<2, true> is the 6th k_scan launch
#    of the driver (warm-up propagate + one measured: <1,false> <2,false> <2,true> each; the heavy pass 1 is off)
for spec in "k_compress 1 k_compress" "k_scan 5 k_scan2true"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k $1 --launch-skip $2 --launch-count 1 \
      -o $O/full_c4_$3 -f python tools/ncu_driver.py c4 1 256 > $O/full_c4_$3.log 2>&1
  echo "full $3 rc=$?"
  ncu -i $O/full_c4_$3.ncu-rep --page raw --csv > $O/full_c4_$3.csv 2>/dev/null
  rm -f $O/full_c4_$3.ncu-rep
done
# 5. GPU test log
python -m pytest tests -m gpu -q > $O/gputest.log 2>&1; echo "pytest rc=$?" >> $O/gputest.log; tail -2 $O/gputest.log
python -m pytest tests/test_gpu_scale.py -q -s 2>&1 | grep -E "^c[0-9]|passed|failed" > $O/scale_parity.log
true
