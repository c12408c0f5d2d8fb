# after the parallel partial-sum loads and the deeper ghost prefetch: configs 2 / 3 / 5 + traces
mkdir -p gpurun_out
for w in c2 c3 c5; do
  python bench.py --workload $w --steps 5 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/abD_${w}.json 2> gpurun_out/abD_${w}.err
  python -c "
import json; d=json.loads(open('gpurun_out/abD_${w}.json').read().strip().splitlines()[-1])
t=d['timings']; print('$w', round(d['value']/1e6,3), round(d['ms_per_step'],2), 'local', round(t['local_s']*1e3,2), 'strip', round(t['iface_s']*1e3,2), 'aug', round(t['aug_s']*1e3,2), 'setup', round(t['setup_s'],4), t.get('local_cg_iterations'), t.get('strip_cg_iterations'), {k:(v['kernel'], round(v['frac'],3)) for k,v in d['rooflines'].items()}, d['config']['lambdas'][:2])"
done
MLG_RES_TRACE=1 python bench.py --workload c2 --steps 1 --warmup 0 --no-extras --no-cpu-baseline 2>&1 | grep "resident trace" | tail -2 > gpurun_out/resident_trace_c2_r2D.txt; cat gpurun_out/resident_trace_c2_r2D.txt
MLG_RES_TRACE=1 python bench.py --workload c5 --steps 1 --warmup 0 --no-extras --no-cpu-baseline 2>&1 | grep "resident trace" | tail -1
