# resident selection rule (batches beyond L2): config 3 and config 2 timings + L-shape / path tests
TAG=${1:-r2k2}
mkdir -p gpurun_out
for w in c3 c2; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/sel_${w}_$TAG.json 2> gpurun_out/sel_${w}_$TAG.err; echo "$w rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/sel_${w}_$TAG.json').read().splitlines()[-1]);print('$w', d['value'], d['timings'], d['config']['lambdas'], {k:(v['kernel'], v['bound'], round(v['frac'],3)) for k,v in d['rooflines'].items()})"
done
timeout 1500 python -m pytest tests/test_gpu_lshape.py tests/test_gpu_cg_paths.py tests/test_gpu_solvers.py tests/test_gpu_bench.py -q -x > gpurun_out/pt_$TAG.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pt_$TAG.log
