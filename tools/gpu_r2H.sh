# tile height of the config-5 strip solve (MLG_CG_STRIP_ROWS) against the automatic choice
mkdir -p gpurun_out
for r in ${ROWS:-0 32 48 64 80 96 128}; do
  MLG_CG_STRIP_ROWS=$r python bench.py --workload c5 --steps 2 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/abrows_$r.json 2> gpurun_out/abrows_$r.err
  python -c "
import json; d=json.loads(open('gpurun_out/abrows_$r.json').read().strip().splitlines()[-1])
t=d['timings']; print('strip_rows=$r', round(d['value']/1e6,3), round(d['ms_per_step'],2), 'local', round(t['local_s']*1e3,2), 'strip', round(t['iface_s']*1e3,2), t.get('strip_cg_iterations'), d['rooflines']['strip']['launches'])"
done
