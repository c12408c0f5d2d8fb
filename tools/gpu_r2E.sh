# fused boundary-row publish (default) against the separate pass (ab/libmlg_nofuse.so):
# small golden case, configs 2 and 5, traces
mkdir -p gpurun_out
for v in default ${VARIANTS:-nofuse}; do
  if [ $v = default ]; then L=""; else L="MLG_LIB=ab/libmlg_$v.so"; fi
  env $L timeout 300 python tools/sanitize_case.py resident > gpurun_out/small_${v}_r2E.log 2>&1; echo "small $v rc=$?"
  for w in ${WL:-c2 c5}; do
    env $L python bench.py --workload $w --steps 5 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/abE_${v}_${w}.json 2> gpurun_out/abE_${v}_${w}.err
    python -c "
import json; d=json.loads(open('gpurun_out/abE_${v}_${w}.json').read().strip().splitlines()[-1])
t=d['timings']; print('$v $w', round(d['value']/1e6,3), round(d['ms_per_step'],2), 'local', round(t['local_s']*1e3,2), 'strip', round(t['iface_s']*1e3,2), 'setup', round(t['setup_s'],4), t.get('local_cg_iterations'), t.get('strip_cg_iterations'), d['config']['lambdas'][:2])"
    env $L MLG_RES_TRACE=1 python bench.py --workload $w --steps 1 --warmup 0 --no-extras --no-cpu-baseline 2>&1 | grep "resident trace" | tail -2 > gpurun_out/resident_trace_${w}_${v}_r2E.txt; cat gpurun_out/resident_trace_${w}_${v}_r2E.txt
  done
done
