#!/bin/bash
# Propagate phase times (bench loop, L2 flushed) of configs without the oracle legs:
#   CONFIGS="c4 c5" bash tools/quick_bench.sh
for cfg in ${CONFIGS:-c4}; do
  python bench.py --config $cfg --parity off --no-cpu-baseline --e2e-steps 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$cfg', 'propagate', round(d['ms_per_step'],3), {k:round(v['ms'],3) for k,v in d['roofline'].get('phases',{}).items()}, 'e2e', round(d['e2e']['k_seed_wall_s']*1e3,2), d['e2e']['step_phase_ms'][-1])
"
done
