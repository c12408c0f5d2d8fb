for cfg in "8192 16" "16384 4" "16384 8" "32768 4" "4096 32"; do
  set -- $cfg
  MLG_CG_TASKS=$1 MLG_CG_MINROWS=$2 python bench.py --no-cpu-baseline > gpurun_out/sw_$1_$2.json 2>/dev/null
  python -c "
import json,sys; d=json.loads(open('gpurun_out/sw_$1_$2.json').read().strip().splitlines()[-1]); ns=d['north_star_workload']
print('$1 $2', round(d['value']/1e6,2), round(d['ms_per_step'],2), round(d['timings']['local_s']*1e3,1), round(d['timings']['iface_s']*1e3,1), '| c5', round(ns['value']/1e6,3), round(ns['timings']['local_s'],3), round(ns['timings']['iface_s'],3))"
done
