# resident CG v3 (counter barrier, 2 CTAs/SM): A/B vs 512-thread CTAs at config 5, GPU tests
TAG=${1:-r2g}
mkdir -p gpurun_out
C5="python bench.py --workload c5 --steps 2 --warmup 1 --no-extras --no-cpu-baseline"
for v in default t512; do
  if [ $v = default ]; then L=""; else L="MLG_LIB=ab/libmlg_$v.so"; fi
  env $L MLG_RES_TRACE=1 $C5 > gpurun_out/ab_${v}_$TAG.json 2> gpurun_out/ab_${v}_$TAG.err; echo "$v rc=$?"; grep "resident trace" gpurun_out/ab_${v}_$TAG.err | tail -1
  python -c "import json;d=json.loads(open('gpurun_out/ab_${v}_$TAG.json').read().splitlines()[-1]);print('$v', d['value'], d['timings'])"
done
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pt_$TAG.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pt_$TAG.log
