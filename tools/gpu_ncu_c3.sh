# ncu --set full of the L-shape (config 3) local-solve k_cg_iter on the
# constant-coefficient async path (hole excluded by geometry).
TAG=${1:-r1}
mkdir -p gpurun_out
C3="python bench.py --workload c3 --steps 1 --warmup 0 --no-north-star --no-cpu-baseline"
$C3 > gpurun_out/plain_c3.log 2>&1 || { echo plain c3 failed; tail gpurun_out/plain_c3.log; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_c3_$TAG.csv $C3 > gpurun_out/ncu_launch_c3.log 2>&1; echo ncu_launch rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_cg_iter' -s 400 -c 2 -o gpurun_out/prof_iter_c3_$TAG $C3 > gpurun_out/ncu_c3.log 2>&1; echo ncu_c3 rc=$?
