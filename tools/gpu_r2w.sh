# full GPU suite + bench line (all workloads) at HEAD; copies go to profiles/
TAG=${1:-r2w}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_$TAG.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/gpu_tests_$TAG.log
timeout 1500 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?
python -c "import json;d=json.loads(open('gpurun_out/bench_$TAG.json').read().splitlines()[-1]);print(d['value'], d['e2e']['value'], d['timings']); print({k:(v['kernel'], round(v['frac'],3)) for k,v in d['rooflines'].items()})"
