# resident CG v1 sync + chunked phases: A/B at config 5 (trace)
TAG=${1:-r2h}
mkdir -p gpurun_out
C5="python bench.py --workload c5 --steps 2 --warmup 1 --no-extras --no-cpu-baseline"
for v in default t256 c8; do
  if [ $v = default ]; then L=""; else L="MLG_LIB=ab/libmlg_$v.so"; fi
  env $L MLG_RES_TRACE=1 $C5 > gpurun_out/ab_${v}_$TAG.json 2> gpurun_out/ab_${v}_$TAG.err; echo "$v rc=$?"; grep "resident trace" gpurun_out/ab_${v}_$TAG.err | tail -1
  python -c "import json;d=json.loads(open('gpurun_out/ab_${v}_$TAG.json').read().splitlines()[-1]);print('$v', d['value'], d['timings']['local_s'], d['timings']['iface_s'])"
done
