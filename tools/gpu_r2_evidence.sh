# Resident trace at config 5, ncu --set full of the three config-5 kernels
# (L7 local k_cg_resident, L7 strip k_cg_iter pair, L7 k_assemble), and
# compute-sanitizer on the small multilevel case through each CG kernel.
TAG=${1:-r2e}
mkdir -p gpurun_out
C5="python bench.py --workload c5 --steps 1 --warmup 0 --no-extras --no-cpu-baseline"
MLG_RES_TRACE=1 $C5 > gpurun_out/trace_$TAG.json 2> gpurun_out/trace_$TAG.err; echo trace rc=$?; grep "resident trace" gpurun_out/trace_$TAG.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_assemble -s 7 -c 1 -o gpurun_out/prof_asm_c5_$TAG $C5 > gpurun_out/ncu_asm_$TAG.log 2>&1; echo ncu_asm rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cg_iter -s 6000 -c 2 -o gpurun_out/prof_strip_c5_$TAG $C5 > gpurun_out/ncu_strip_$TAG.log 2>&1; echo ncu_strip rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_cg_resident -s 3 -c 1 -o gpurun_out/prof_res_c5_$TAG $C5 > gpurun_out/ncu_res_$TAG.log 2>&1; echo ncu_res rc=$?
for mode in resident persist iter; do
  for tool in memcheck racecheck synccheck; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py $mode > gpurun_out/san_${mode}_${tool}_$TAG.log 2>&1; echo "san $mode $tool rc=$?"; tail -1 gpurun_out/san_${mode}_${tool}_$TAG.log
  done
done
