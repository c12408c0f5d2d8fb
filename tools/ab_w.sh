# A/B of any workload: tools/ab_w.sh WORKLOAD name[@ENV=VAL,...] ...
W=$1; shift
for spec in "$@"; do
  v=${spec%@*}
  envs=""
  [ "$spec" != "$v" ] && envs=$(echo ${spec#*@} | tr ',' ' ')
  tag=$(echo "$spec" | tr '@=,' '___')
  env $envs MLG_LIB=$PWD/ab/libmlg_$v.so timeout 600 python bench.py --workload $W --no-north-star --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/abw_${W}_$tag.json 2>gpurun_out/abw_${W}_$tag.err
  python -c "
import json; d=json.loads(open('gpurun_out/abw_${W}_$tag.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$W $spec', round(d['value']/1e6,3), round(d['ms_per_step'],1), 'local', round(d['timings']['local_s'],4), 'strip', round(d['timings']['iface_s'],4), 'avg_launch_ms', round(r['avg_launch_ms'],4), 'frac', round(r['frac'],3), 'lam', d['config'].get('lambdas'))"
done
