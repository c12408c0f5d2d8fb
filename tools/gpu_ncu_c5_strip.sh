# Launch list of one config-5 step (k_cg_iter only) and an ncu --set full
# capture of a strip-solve launch (found by its grid size in the list).
export TAG=${1:-r1}
mkdir -p gpurun_out
C5="python bench.py --workload c5 --steps 1 --warmup 0 --no-cpu-baseline --no-north-star"
$C5 > gpurun_out/plain_c5s.log 2>&1 || { echo plain failed; tail gpurun_out/plain_c5s.log; exit 1; }
timeout 1500 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -k regex:k_cg_iter --csv --log-file gpurun_out/launches_c5_$TAG.csv $C5 > gpurun_out/ncu_l5.log 2>&1; echo list rc=$?
python - <<'PY'
import csv
import os
rows=list(csv.reader(open('gpurun_out/launches_c5_%s.csv' % os.environ['TAG'])))
h=[i for i,r in enumerate(rows) if 'ID' in r][0]; hdr=rows[h]
idx=hdr.index('ID'); mn=hdr.index('Metric Name'); mv=hdr.index('Metric Value')
grid={}; dur={}
for r in rows[h+1:]:
    if len(r)<=mv: continue
    i=int(r[idx])
    if r[mn]=='launch__grid_size': grid[i]=r[mv]
    if r[mn]=='gpu__time_duration.sum': dur[i]=float(r[mv].replace(',',''))
n=len(grid); last=max(grid)
# the last ~2400 launches of the run are the level-7 strip solve (4 systems, one window)
g_last=grid[last]
first_strip=min(i for i in grid if grid[i]==g_last and i>last-3000)
print("launches",n,"last grid",g_last,"first strip-like id",first_strip)
open('gpurun_out/strip_skip.txt','w').write(str(first_strip+200))
PY
SKIP=$(cat gpurun_out/strip_skip.txt)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cg_iter -s $SKIP -c 1 -o gpurun_out/prof_iter_c5_strip_$TAG $C5 > gpurun_out/ncu_c5s.log 2>&1; echo full rc=$?
