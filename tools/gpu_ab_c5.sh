# config-5 A/B of libraries built by tools/build_ab.py: small case, plain timing (2 steps)
# and one traced step per variant
TAG=${1:-ab}; shift
mkdir -p gpurun_out
C5="python bench.py --workload c5 --steps 2 --warmup 1 --no-extras --no-cpu-baseline"
for v in default "$@"; do
  if [ $v = default ]; then L=""; else L="MLG_LIB=ab/libmlg_$v.so"; fi
  env $L timeout 300 python tools/sanitize_case.py resident > gpurun_out/small_${v}_$TAG.log 2>&1; echo "small $v rc=$?"
  env $L timeout 600 $C5 > gpurun_out/ab_${v}_$TAG.json 2> gpurun_out/ab_${v}_$TAG.err; echo "$v rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/ab_${v}_$TAG.json').read().splitlines()[-1]);print('$v', d['value'], d['timings']['local_s'], d['timings']['iface_s'], d['config']['lambdas'])"
  env $L MLG_RES_TRACE=1 timeout 600 python bench.py --workload c5 --steps 1 --warmup 0 --no-extras --no-cpu-baseline > gpurun_out/trace_${v}_$TAG.json 2> gpurun_out/trace_${v}_$TAG.err; grep "resident trace" gpurun_out/trace_${v}_$TAG.err | grep "3 lanes" | tail -1
done
