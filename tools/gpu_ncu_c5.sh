# ncu --set full of one local-solve and one strip-solve k_cg_iter launch at config 5
TAG=${1:-r1}
C5="python bench.py --workload c5 --steps 1 --warmup 0 --no-cpu-baseline"
$C5 > gpurun_out/plain_c5.log 2>&1 || { echo plain failed; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:'k_cg_iter' -s 5500 -c 1 -o gpurun_out/prof_iter_c5_local_$TAG $C5 > gpurun_out/ncu_c5a.log 2>&1; echo ncu1 rc=$?
ncu --set full --clock-control none --import-source on -k regex:'k_cg_iter' -s 8000 -c 1 -o gpurun_out/prof_iter_c5_strip_$TAG $C5 > gpurun_out/ncu_c5b.log 2>&1; echo ncu2 rc=$?
