# ncu --set full of the level-7 local k_cg_resident launch at config 5
TAG=${1:-r2j}
mkdir -p gpurun_out
C5="python bench.py --workload c5 --steps 1 --warmup 0 --no-extras --no-cpu-baseline"
$C5 > gpurun_out/plain_$TAG.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cg_resident -s 9 -c 1 -o gpurun_out/prof_res_L7_$TAG $C5 > gpurun_out/ncu_$TAG.log 2>&1; echo ncu rc=$?; tail -2 gpurun_out/ncu_$TAG.log
