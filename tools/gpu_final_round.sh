# Round-end evidence at HEAD: full GPU tests, smoke, default bench line, c4 ncu
# of the general-stencil k_cg_iter (flag-free interior sweep), c2 launch list.
TAG=${1:-r1}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pt_$TAG.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pt_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke rc=$?
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?
C4="python bench.py --workload c4 --steps 1 --warmup 0 --no-north-star --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_cg_iter' -s 3000 -c 1 -o gpurun_out/prof_iter_c4_$TAG $C4 > gpurun_out/ncu_c4.log 2>&1; echo ncu_c4 rc=$?
LIGHT="python bench.py --steps 1 --warmup 1 --no-north-star --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_c2_$TAG.csv $LIGHT > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch rc=$?
