# costly tiles first in the per-iteration launches (MLG_CG_LPT=1, default) against the
# system-major order (0): configs 5 and 4
mkdir -p gpurun_out
for w in c5 c4; do for m in 0 1 0 1; do
  MLG_CG_LPT=$m python bench.py --workload $w --steps 3 --warmup 2 --no-extras --no-cpu-baseline > gpurun_out/ablpt_${w}_$m.json 2> gpurun_out/ablpt_${w}_$m.err
  python -c "
import json; d=json.loads(open('gpurun_out/ablpt_${w}_$m.json').read().strip().splitlines()[-1])
t=d['timings']; print('$w lpt=$m', round(d['value']/1e6,3), round(d['ms_per_step'],2), 'local', round(t['local_s']*1e3,2), 'strip', round(t['iface_s']*1e3,2), t.get('local_cg_iterations'), t.get('strip_cg_iterations'), d['config']['lambdas'][:2])"
done; done
