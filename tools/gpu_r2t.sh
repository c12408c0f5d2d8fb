TAG=${1:-r2t}; shift
mkdir -p gpurun_out
timeout 300 python tools/sanitize_case.py resident > gpurun_out/small_$TAG.log 2>&1; echo small rc=$?; tail -1 gpurun_out/small_$TAG.log
C5="python bench.py --workload c5 --steps 1 --warmup 1 --no-extras --no-cpu-baseline"
for v in default "$@"; do
  if [ $v = default ]; then L=""; else L="MLG_LIB=ab/libmlg_$v.so"; fi
  env $L MLG_RES_TRACE=1 timeout 600 $C5 > gpurun_out/ab_${v}_$TAG.json 2> gpurun_out/ab_${v}_$TAG.err; echo "$v rc=$?"; grep "resident trace" gpurun_out/ab_${v}_$TAG.err | grep "3 lanes\|local" | tail -1
  python -c "import json;d=json.loads(open('gpurun_out/ab_${v}_$TAG.json').read().splitlines()[-1]);print('$v', d['value'], d['timings']['local_s'], d['timings']['iface_s'], d['config']['lambdas'])"
done
