# ncu --set full of the general-stencil k_cg_iter at config 4 (reaction field), level-7 local
# solves: the launch is found by its grid size in a launch list of the same command.
export TAG=${1:-r2}
mkdir -p gpurun_out
C4="python bench.py --workload c4 --steps 1 --warmup 0 --no-extras --no-cpu-baseline"
$C4 > gpurun_out/plain_c4.log 2>&1 || { echo plain c4 failed; tail gpurun_out/plain_c4.log; exit 1; }
timeout 1200 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -k regex:k_cg_iter --csv --log-file gpurun_out/launches_c4_$TAG.csv $C4 > gpurun_out/ncu_l4.log 2>&1; echo list rc=$?
python - <<'PY'
import csv, os
rows=list(csv.reader(open('gpurun_out/launches_c4_%s.csv' % os.environ['TAG'])))
h=[i for i,r in enumerate(rows) if 'ID' in r][0]; hdr=rows[h]
idx=hdr.index('ID'); mn=hdr.index('Metric Name'); mv=hdr.index('Metric Value')
grid={}
for r in rows[h+1:]:
    if len(r)<=mv: continue
    if r[mn]=='launch__grid_size': grid[int(r[idx])]=int(r[mv].replace(',',''))
ids=sorted(grid); gmax=max(grid.values())
first=[k for k,i in enumerate(ids) if grid[i]==gmax][0]
print("k_cg_iter launches", len(ids), "largest grid", gmax, "first at position", first)
open('gpurun_out/c4_skip.txt','w').write(str(first+200))
PY
SKIP=$(cat gpurun_out/c4_skip.txt)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cg_iter -s $SKIP -c 1 -o gpurun_out/prof_iter_c4_$TAG $C4 > gpurun_out/ncu_c4.log 2>&1; echo ncu_c4 rc=$?
