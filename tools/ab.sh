for v in "$@"; do
  MLG_LIB=$PWD/ab/libmlg_$v.so python bench.py --no-cpu-baseline > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]); ns=d['north_star_workload']
print('$v', round(d['value']/1e6,3), round(d['ms_per_step'],2), round(d['timings']['local_s']*1e3,2), round(d['timings']['iface_s']*1e3,2), '| c5', round(ns['value']/1e6,3), round(ns['timings']['local_s'],3), round(ns['timings']['iface_s'],3))"
done
