set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
python bench.py > gpurun_out/bench_r1a.json 2> gpurun_out/bench_r1a.err; echo bench rc=$?
tail -c 3000 gpurun_out/bench_r1a.json
LIGHT="python bench.py --steps 1 --warmup 1 --no-north-star --no-cpu-baseline"
$LIGHT > gpurun_out/plain_c2.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c2.csv $LIGHT > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
$LIGHT > gpurun_out/plain_c2b.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_cg_a -s 300 -c 2 -o gpurun_out/prof_ka_c2 $LIGHT > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
C5="python bench.py --workload c5 --steps 1 --warmup 0 --no-cpu-baseline"
$C5 > gpurun_out/plain_c5.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_cg_a -s 5600 -c 2 -o gpurun_out/prof_ka_c5 $C5 > gpurun_out/ncu_full_c5.log 2>&1; echo ncu3 rc=$?
ls -la gpurun_out/
