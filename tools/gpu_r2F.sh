# Round-2 final evidence at HEAD: reference arm (config 5, box-measured), GPU tests, the
# driver's bench line, resident traces (configs 5 and 2), launch list, ncu --set full of
# k_cg_resident at config 5 (local solves) and config 2 (local + strip launches of level 6).
TAG=${1:-r2F}
mkdir -p gpurun_out
( time timeout 1500 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/refarm_$TAG.json 2> gpurun_out/refarm_$TAG.err ) 2> gpurun_out/refarm_time_$TAG.txt; echo ref rc=$?; tail -3 gpurun_out/refarm_time_$TAG.txt
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_$TAG.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/gpu_tests_$TAG.log
( time timeout 1500 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err ) 2> gpurun_out/bench_time_$TAG.txt; echo bench rc=$?; tail -3 gpurun_out/bench_time_$TAG.txt
python -c "import json;d=json.loads(open('gpurun_out/bench_$TAG.json').read().splitlines()[-1]);print(d['value'], d['e2e']['value'], d['timings'], d['cpu_baseline']['value']); print({k:(v['kernel'], round(v['frac'],3)) for k,v in d['rooflines'].items()}); print({k:d[k]['value'] for k in d if k.endswith('_workload')})"
C5="python bench.py --workload c5 --steps 1 --warmup 0 --no-extras --no-cpu-baseline"
C2="python bench.py --workload c2 --steps 1 --warmup 0 --no-extras --no-cpu-baseline"
MLG_RES_TRACE=1 $C5 > gpurun_out/trace_$TAG.json 2> gpurun_out/trace_$TAG.err; grep "resident trace" gpurun_out/trace_$TAG.err | grep "3 lanes" | tail -1 > gpurun_out/resident_trace_c5_$TAG.txt; cat gpurun_out/resident_trace_c5_$TAG.txt
MLG_RES_TRACE=1 $C2 2>&1 | grep "resident trace" | tail -2 > gpurun_out/resident_trace_c2_$TAG.txt; cat gpurun_out/resident_trace_c2_$TAG.txt
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5_$TAG.csv $C5 > gpurun_out/ncu_launches_$TAG.log 2>&1; echo launches rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_$TAG.csv $C2 > gpurun_out/ncu_launches_c2_$TAG.log 2>&1; echo launches c2 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cg_resident -s 1 -c 2 -o gpurun_out/prof_res_c2_$TAG $C2 > gpurun_out/ncu_res_c2_$TAG.log 2>&1; echo ncu_res_c2 rc=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_cg_resident -s 7 -c 1 -o gpurun_out/prof_res_c5_$TAG $C5 > gpurun_out/ncu_res_$TAG.log 2>&1; echo ncu_res rc=$?
