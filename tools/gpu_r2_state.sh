# Session-start evidence at HEAD: GPU tests, smoke, default bench line, c5 launch list
TAG=${1:-r2s}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke rc=$?
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?
timeout 1800 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/pt_$TAG.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pt_$TAG.log
C5="python bench.py --workload c5 --steps 1 --warmup 0 --no-extras --no-cpu-baseline"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/launches_c5_$TAG.csv $C5 > gpurun_out/ncu_launch_$TAG.log 2>&1; echo ncu_launch rc=$?
