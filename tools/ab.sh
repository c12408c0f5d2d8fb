# A/B of library variants built by tools/build_ab.py: tools/ab.sh name[@ENV=VAL] ...
for spec in "$@"; do
  v=${spec%@*}
  envs=""
  [ "$spec" != "$v" ] && envs=${spec#*@}
  tag=$(echo "$spec" | tr '@=' '__')
  env $envs MLG_LIB=$PWD/ab/libmlg_$v.so python bench.py --no-cpu-baseline > gpurun_out/ab_$tag.json 2>gpurun_out/ab_$tag.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$tag.json').read().strip().splitlines()[-1]); ns=d['north_star_workload']
print('$spec', round(d['value']/1e6,3), round(d['ms_per_step'],2), round(d['timings']['local_s']*1e3,2), round(d['timings']['iface_s']*1e3,2), '| c5', round(ns['value']/1e6,3), round(ns['timings']['local_s'],3), round(ns['timings']['iface_s'],3))"
done
