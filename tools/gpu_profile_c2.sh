# Config-2 profile evidence at HEAD: launch list of one step and ncu --set full
# of the persistent CG launches (warm L2).
TAG=${1:-r1}
mkdir -p gpurun_out
LIGHT="python bench.py --steps 1 --warmup 1 --no-north-star --no-cpu-baseline"
$LIGHT > gpurun_out/plain_c2.log 2>&1 || { echo plain c2 failed; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_c2_$TAG.csv $LIGHT > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch rc=$?
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:'k_cg_persist' -s 8 -c 2 -o gpurun_out/prof_persist_c2_$TAG $LIGHT > gpurun_out/ncu_p.log 2>&1; echo ncu_c2 rc=$?
