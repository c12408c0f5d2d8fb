# assembly with the per-level table + reference arm wall time at config 5
TAG=${1:-r2x}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_structure.py tests/test_gpu_lshape.py -q -x > gpurun_out/pt_$TAG.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pt_$TAG.log
python bench.py --workload c5 --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?
python -c "import json;d=json.loads(open('gpurun_out/bench_$TAG.json').read().splitlines()[-1]);print(d['value'], d['timings']); a=d['rooflines']['assembly']; print(a['kernel'], a['avg_launch_ms'], a['frac'])"
nproc
( time timeout 1500 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/refarm_$TAG.json 2> gpurun_out/refarm_$TAG.err ) 2> gpurun_out/refarm_time_$TAG.txt; echo ref rc=$?; cat gpurun_out/refarm_time_$TAG.txt; head -c 1500 gpurun_out/refarm_$TAG.json
