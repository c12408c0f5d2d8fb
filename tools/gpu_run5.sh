python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_arm.json 2> gpurun_out/ref_arm.err; echo ref rc=$?
tail -c 1500 gpurun_out/ref_arm.json
C5="python bench.py --workload c5 --steps 1 --warmup 0 --no-cpu-baseline"
$C5 > gpurun_out/plain_c5.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:'k_cg_iter' -s 5500 -c 1 -o gpurun_out/prof_iter_c5_local_v3 $C5 > gpurun_out/ncu_c5a.log 2>&1; echo ncu1 rc=$?
ncu --set full --clock-control none --import-source on -k regex:'k_cg_iter' -s 8000 -c 1 -o gpurun_out/prof_iter_c5_strip_v3 $C5 > gpurun_out/ncu_c5b.log 2>&1; echo ncu2 rc=$?
LIGHT="python bench.py --steps 1 --warmup 1 --no-north-star --no-cpu-baseline"
$LIGHT > gpurun_out/plain_c2.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 5000 -c 3000 --csv --log-file gpurun_out/launches_c2_v3.csv $LIGHT > gpurun_out/ncu_launch.log 2>&1; echo ncu3 rc=$?
ncu --set full --clock-control none --import-source on -k regex:'k_cg_iter' -s 3000 -c 1 -o gpurun_out/prof_iter_c2_v3 $LIGHT > gpurun_out/ncu_c2.log 2>&1; echo ncu4 rc=$?
