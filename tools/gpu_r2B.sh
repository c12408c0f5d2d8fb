# A/B: SM-resident CG forced wherever it fits (MLG_CG_RESIDENT=2) against the default kernel
# choice, configs 2 / 3 / 4; resident phase trace of the config-2 run.
mkdir -p gpurun_out
for w in c2 c3 c4; do for m in 1 2; do
  MLG_CG_RESIDENT=$m python bench.py --workload $w --steps 5 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/abres_${w}_$m.json 2> gpurun_out/abres_${w}_$m.err
  python -c "
import json; d=json.loads(open('gpurun_out/abres_${w}_$m.json').read().strip().splitlines()[-1])
t=d['timings']; print('$w resident=$m', round(d['value']/1e6,3), round(d['ms_per_step'],2), 'local', round(t['local_s']*1e3,2), 'strip', round(t['iface_s']*1e3,2), 'aug', round(t['aug_s']*1e3,2), t.get('local_cg_iterations'), t.get('strip_cg_iterations'), {k:(v['kernel'], round(v['frac'],3)) for k,v in d['rooflines'].items()})"
done; done
MLG_CG_RESIDENT=2 MLG_RES_TRACE=1 python bench.py --workload c2 --steps 1 --warmup 0 --no-extras --no-cpu-baseline 2>&1 | grep "resident trace" | tail -4
# alternating tile order of the HBM-streaming strip solve (config 5), and config 4's streaming batches
for w in c5 c4; do for m in 0 1 0 1; do
  MLG_CG_BOUSTRO=$m python bench.py --workload $w --steps 3 --warmup 2 --no-extras --no-cpu-baseline > gpurun_out/abbou_${w}_$m.json 2> gpurun_out/abbou_${w}_$m.err
  python -c "
import json; d=json.loads(open('gpurun_out/abbou_${w}_$m.json').read().strip().splitlines()[-1])
t=d['timings']; print('$w boustro=$m', round(d['value']/1e6,3), round(d['ms_per_step'],2), 'local', round(t['local_s']*1e3,2), 'strip', round(t['iface_s']*1e3,2), t.get('local_cg_iterations'), t.get('strip_cg_iterations'), d['config']['lambdas'][:2])"
done; done
timeout 900 python -m pytest tests/test_gpu_north_star.py -x -q -k "strip_iterations or local_iterations" 2>&1 | tail -5
