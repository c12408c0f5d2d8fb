# Round profile evidence: bench line, C2 launch list, ncu --set full of the
# dominant CG kernels at config 2 (persistent, warm L2) and config 5 (async).
TAG=${1:-r1}
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?
LIGHT="python bench.py --steps 1 --warmup 1 --no-north-star --no-cpu-baseline"
$LIGHT > gpurun_out/plain_c2.log 2>&1 || { echo plain c2 failed; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_c2_$TAG.csv $LIGHT > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch rc=$?
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:'k_cg_persist' -s 8 -c 2 -o gpurun_out/prof_persist_c2_$TAG $LIGHT > gpurun_out/ncu_p.log 2>&1; echo ncu_c2 rc=$?
C5="python bench.py --workload c5 --steps 1 --warmup 0 --no-cpu-baseline"
$C5 > gpurun_out/plain_c5.log 2>&1 || { echo plain c5 failed; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_cg_iter' -s 5500 -c 1 -o gpurun_out/prof_iter_c5_local_$TAG $C5 > gpurun_out/ncu_c5a.log 2>&1; echo ncu_c5 rc=$?
