# ncu --set full of the general-stencil k_cg_iter (config 4, reaction field) and
# of the arrowhead augmented kernel (config 2), for the round's profile evidence.
TAG=${1:-r1}
mkdir -p gpurun_out
C4="python bench.py --workload c4 --steps 1 --warmup 0 --no-north-star --no-cpu-baseline"
$C4 > gpurun_out/plain_c4.log 2>&1 || { echo plain c4 failed; tail gpurun_out/plain_c4.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_cg_iter' -s 3000 -c 1 -o gpurun_out/prof_iter_c4_$TAG $C4 > gpurun_out/ncu_c4.log 2>&1; echo ncu_c4 rc=$?
LIGHT="python bench.py --steps 1 --warmup 1 --no-north-star --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_aug_arrow|k_errors' -c 2 -o gpurun_out/prof_aug_c2_$TAG $LIGHT > gpurun_out/ncu_aug.log 2>&1; echo ncu_aug rc=$?
