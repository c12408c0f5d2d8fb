# A/B of the config-5 CG launch time: tools/ab_c5.sh name[@ENV=VAL,...] ...
for spec in "$@"; do
  v=${spec%@*}
  envs=""
  [ "$spec" != "$v" ] && envs=$(echo ${spec#*@} | tr ',' ' ')
  tag=$(echo "$spec" | tr '@=,' '___')
  env $envs MLG_LIB=$PWD/ab/libmlg_$v.so timeout 600 python bench.py --workload c5 --no-north-star --no-cpu-baseline --steps 1 --warmup 1 > gpurun_out/ab5_$tag.json 2>gpurun_out/ab5_$tag.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab5_$tag.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$spec', round(d['value']/1e6,3), round(d['ms_per_step'],1), 'local', round(d['timings']['local_s'],3), 'strip', round(d['timings']['iface_s'],3), 'avg_launch_ms', round(r['avg_launch_ms'],4), 'frac', round(r['frac'],3), 'its', d['timings']['local_cg_iterations'])"
done
