# A/B of config-2 step time: tools/ab_c2.sh name[@ENV=VAL,ENV=VAL] ...
for spec in "$@"; do
  v=${spec%@*}
  envs=""
  [ "$spec" != "$v" ] && envs=$(echo ${spec#*@} | tr ',' ' ')
  tag=$(echo "$spec" | tr '@=,' '___')
  env $envs MLG_LIB=$PWD/ab/libmlg_$v.so python bench.py --no-north-star --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/ab_$tag.json 2>gpurun_out/ab_$tag.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$tag.json').read().strip().splitlines()[-1])
print('$spec', round(d['value']/1e6,3), round(d['ms_per_step'],2), round(d['timings']['local_s']*1e3,2), round(d['timings']['iface_s']*1e3,2), round(d['timings']['aug_s']*1e3,2))"
done
