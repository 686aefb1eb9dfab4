#!/bin/bash
# Per-config ncu metrics of one propagate (after an L2 flush):
#   time, DRAM bytes, L2 sectors by op (read / atomic / reduction / write)
# -> gpurun_out/ncu_<cfg>.csv ; summarise with tools/ncu_summarize.py <cfg> ...
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_atom.sum,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum
for cfg in ${CONFIGS:-c1 c2 c2p1 c3 c4 c5}; do
  timeout 1200 ncu --replay-mode application --metrics $M --clock-control none --csv --print-units base \
      --log-file gpurun_out/ncu_$cfg.csv python tools/ncu_driver.py $cfg 1 > gpurun_out/ncu_$cfg.log 2>&1
  echo "$cfg rc=$?"
done
