# resident CG: correctness (GPU tests), trace of the c2 step, ncu of one resident launch
TAG=${1:-r2d}
mkdir -p gpurun_out
C2="python bench.py --workload c2 --steps 1 --warmup 3 --no-extras --no-cpu-baseline"
MLG_RES_TRACE=1 $C2 > gpurun_out/trace_$TAG.json 2> gpurun_out/trace_$TAG.err; echo trace rc=$?; grep "resident trace" gpurun_out/trace_$TAG.err | head -8
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pt_$TAG.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pt_$TAG.log
$C2 > gpurun_out/plain_$TAG.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cg_resident -s 2 -c 2 -o gpurun_out/prof_res_c2_$TAG $C2 > gpurun_out/ncu_$TAG.log 2>&1; echo ncu rc=$?
