IMX_PULL_TILE=1 IMX_HOOK=pull timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for t in 0 1; do IMX_PULL_TILE=$t timeout 300 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/t_c5_$t.json 2>gpurun_out/t_c5_$t.err; python - c5 $t <<'PY'
import json,sys
try:
    d=json.loads(open(f'gpurun_out/t_{sys.argv[1]}_{sys.argv[2]}.json').read().strip().splitlines()[-1]); r=d['roofline']
    print(sys.argv[1], sys.argv[2], round(d['ms_per_step'],3), {k:round(v,3) for k,v in r['kernel_ms'].items()}, 'e2e', round(d['e2e']['k_seed_wall_s']*1e3,2), d['e2e']['seeds_head'], d['e2e']['spread'])
except Exception as e: print(sys.argv[1:], 'fail', e)
PY
done
