# resident CG at config 5: per-phase trace and ncu of the level-7 local launch
TAG=${1:-r2e}
mkdir -p gpurun_out
C5="python bench.py --workload c5 --steps 1 --warmup 0 --no-extras --no-cpu-baseline"
MLG_RES_TRACE=1 $C5 > gpurun_out/trace_$TAG.json 2> gpurun_out/trace_$TAG.err; echo trace rc=$?; grep "resident trace" gpurun_out/trace_$TAG.err
$C5 > gpurun_out/plain_$TAG.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_cg_resident -c 40 -o gpurun_out/prof_res_c5_$TAG $C5 > gpurun_out/ncu_$TAG.log 2>&1; echo ncu rc=$?; tail -3 gpurun_out/ncu_$TAG.log
