# ncu --set full (warm L2: --cache-control none) of k_cg_iter launches at config 2
TAG=${1:-r1}
LIGHT="python bench.py --steps 1 --warmup 1 --no-north-star --no-cpu-baseline"
$LIGHT > gpurun_out/plain_c2.log 2>&1 || { echo plain failed; exit 1; }
ncu --set full --cache-control none --clock-control none --import-source on -k regex:'k_cg_iter' -s 3000 -c 1 -o gpurun_out/prof_iter_c2_local_$TAG $LIGHT > gpurun_out/ncu_c2a.log 2>&1; echo ncu1 rc=$?
ncu --set full --cache-control none --clock-control none --import-source on -k regex:'k_cg_iter' -s 4200 -c 1 -o gpurun_out/prof_iter_c2_strip_$TAG $LIGHT > gpurun_out/ncu_c2b.log 2>&1; echo ncu2 rc=$?
ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none -s 2500 -c 2500 --csv --log-file gpurun_out/launches_c2_$TAG.csv $LIGHT > gpurun_out/ncu_c2c.log 2>&1; echo ncu3 rc=$?
