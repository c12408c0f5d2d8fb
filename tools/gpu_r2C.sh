# Resident kernel with slab-sized instantiations (points per thread 48/36/28/20/12) and the new
# kernel choice (resident from 256 k pooled rows): configs 2 / 3 / 5 against the earlier rule
# (MLG_CG_RESIDENT=3), traces, then the CG-path and scale tests.
mkdir -p gpurun_out
for w in c2 c3 c5; do for m in 3 1; do
  MLG_CG_RESIDENT=$m python bench.py --workload $w --steps 5 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/abpt_${w}_$m.json 2> gpurun_out/abpt_${w}_$m.err
  python -c "
import json; d=json.loads(open('gpurun_out/abpt_${w}_$m.json').read().strip().splitlines()[-1])
t=d['timings']; print('$w resident=$m', round(d['value']/1e6,3), round(d['ms_per_step'],2), 'local', round(t['local_s']*1e3,2), 'strip', round(t['iface_s']*1e3,2), 'aug', round(t['aug_s']*1e3,2), 'setup', round(t['setup_s'],4), t.get('local_cg_iterations'), t.get('strip_cg_iterations'), {k:(v['kernel'], round(v['frac'],3)) for k,v in d['rooflines'].items()}, d['config']['lambdas'][:2])"
done; done
MLG_RES_TRACE=1 python bench.py --workload c2 --steps 1 --warmup 0 --no-extras --no-cpu-baseline 2>&1 | grep "resident trace" | tail -2 > gpurun_out/resident_trace_c2_r2C.txt; cat gpurun_out/resident_trace_c2_r2C.txt
MLG_RES_TRACE=1 python bench.py --workload c5 --steps 1 --warmup 0 --no-extras --no-cpu-baseline 2>&1 | grep "resident trace" | cut -c1-260
timeout 1500 python -m pytest tests/test_gpu_cg_paths.py tests/test_gpu_scale.py tests/test_gpu_solvers.py tests/test_gpu_cg_edge.py -x -q 2>&1 | tail -5
