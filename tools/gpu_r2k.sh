# resident CG straight-line phases: correctness (small case + north-star tests) + A/B T=512 vs 256x2
TAG=${1:-r2k}
mkdir -p gpurun_out
python tools/sanitize_case.py resident > gpurun_out/small_$TAG.log 2>&1; echo small rc=$?; tail -2 gpurun_out/small_$TAG.log
MLG_LIB=ab/libmlg_t256.so python tools/sanitize_case.py resident > gpurun_out/small256_$TAG.log 2>&1; echo small256 rc=$?; tail -2 gpurun_out/small256_$TAG.log
C5="python bench.py --workload c5 --steps 2 --warmup 1 --no-extras --no-cpu-baseline"
for v in default t256; do
  if [ $v = default ]; then L=""; else L="MLG_LIB=ab/libmlg_$v.so"; fi
  env $L MLG_RES_TRACE=1 $C5 > gpurun_out/ab_${v}_$TAG.json 2> gpurun_out/ab_${v}_$TAG.err; echo "$v rc=$?"; grep "resident trace" gpurun_out/ab_${v}_$TAG.err | tail -1
  python -c "import json;d=json.loads(open('gpurun_out/ab_${v}_$TAG.json').read().splitlines()[-1]);print('$v', d['value'], d['timings']['local_s'], d['timings']['iface_s'], d['config']['lambdas'])"
done
C2="python bench.py --workload c2 --steps 3 --warmup 3 --no-extras --no-cpu-baseline"
for v in default t256; do
  if [ $v = default ]; then L=""; else L="MLG_LIB=ab/libmlg_$v.so"; fi
  env $L $C2 > gpurun_out/abc2_${v}_$TAG.json 2> gpurun_out/abc2_${v}_$TAG.err; echo "c2 $v rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/abc2_${v}_$TAG.json').read().splitlines()[-1]);print('c2 $v', d['value'], d['timings'])"
done
timeout 900 python -m pytest tests/test_gpu_north_star.py tests/test_gpu_cg_edge.py tests/test_gpu_solvers.py -q -x > gpurun_out/pt_$TAG.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pt_$TAG.log
