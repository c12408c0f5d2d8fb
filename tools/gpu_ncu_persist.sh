# ncu --set full of the persistent CG kernel launches (warm L2) at config 2
TAG=${1:-r1}
SKIP=${2:-8}
LIGHT="python bench.py --steps 1 --warmup 0 --no-north-star --no-cpu-baseline"
$LIGHT > gpurun_out/plain_c2.log 2>&1 || { echo plain failed; exit 1; }
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:'k_cg_persist' -s $SKIP -c 2 -o gpurun_out/prof_persist_c2_$TAG $LIGHT > gpurun_out/ncu_p.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_p.log
