# resident kernel forced on the L2-resident workloads (config 2, config 3): A/B against the persistent kernel
TAG=${1:-r2j}
mkdir -p gpurun_out
for w in c2 c3; do
  for m in 1 2; do
    MLG_CG_RESIDENT=$m MLG_RES_TRACE=1 timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/res_${w}_${m}_$TAG.json 2> gpurun_out/res_${w}_${m}_$TAG.err; echo "$w mode $m rc=$?"
    python -c "import json;d=json.loads(open('gpurun_out/res_${w}_${m}_$TAG.json').read().splitlines()[-1]);print('$w', $m, d['value'], d['timings'], d['config']['lambdas'], {k:(v['kernel'], round(v['frac'],3)) for k,v in d['rooflines'].items()})"
    grep "resident trace" gpurun_out/res_${w}_${m}_$TAG.err | tail -2 | cut -c1-200
  done
done
