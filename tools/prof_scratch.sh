V=paper_2008_03095_b200/lib/variants
echo default; timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
echo pull1; IMX_HOOK=pull IMX_PULL_HEAVY=1 timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
echo hybrid3; IMX_HOOK=hybrid IMX_PULL_HEAVY=3 timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
bm() { cfg=$1; shift; for t in "$@"; do v=${t%%:*}; e=${t#*:}; [ "$e" = "$t" ] && e=X=0; lib=$V/libinfuser_b200_$v.so; [ $v = new ] && lib=paper_2008_03095_b200/lib/libinfuser_b200.so; env $e INFUSER_B200_LIB=$lib timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/t_${cfg}_x.json 2>gpurun_out/t_${cfg}_x.err; python - $cfg $t <<'PY'
import json,sys
try:
    d=json.loads(open(f'gpurun_out/t_{sys.argv[1]}_x.json').read().strip().splitlines()[-1]); r=d['roofline']
    print(sys.argv[1], sys.argv[2], round(d['ms_per_step'],4), {k:round(v,4) for k,v in r['kernel_ms'].items()}, 'e2e', round(d['e2e']['k_seed_wall_s']*1e3,3), d['e2e']['seeds_head'])
except Exception as e: print(sys.argv[1:], 'fail', e)
PY
done; }
bm c3 base new
bm c2 new:IMX_HOOK=pull base:IMX_HOOK=pull
bm c2p1 base new
bm c5 base new
bm c1 base new
