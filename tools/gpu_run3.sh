python bench.py > gpurun_out/bench_r1b.json 2> gpurun_out/bench_r1b.err; echo bench rc=$?
LIGHT="python bench.py --steps 1 --warmup 1 --no-north-star --no-cpu-baseline"
$LIGHT > gpurun_out/plain_c2.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 9700 -c 5000 --csv --log-file gpurun_out/launches_c2.csv $LIGHT > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
C5="python bench.py --workload c5 --steps 1 --warmup 0 --no-cpu-baseline"
$C5 > gpurun_out/plain_c5.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:'k_cg_[ab]' -s 5600 -c 4 -o gpurun_out/prof_cg_c5 $C5 > gpurun_out/ncu_full_c5.log 2>&1; echo ncu2 rc=$?
