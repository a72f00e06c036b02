# Dev tool: per-launch durations of the routing kernels (C2, or C3 with $1 == c3), cold
# (ncu's default cache flush) and warm (--cache-control none), last call of each run
for cc in all none; do
timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control $cc -k regex:route --csv python tools/prof_router.py $1 > gpurun_out/ncu_rt.csv 2>&1
python - $cc <<PY
import csv, sys
rows=[r for r in csv.reader(open("gpurun_out/ncu_rt.csv")) if len(r)>10 and r[-1].replace(".","").replace(",","").isdigit()]
print("cache", sys.argv[1], [(r[4].split("(")[0][-22:], r[-1]) for r in rows[-4:]])
PY
done
python tools/prof_router.py $1
