# Dev tool: M = 128 tail tiles on/off -- tensor-pipe active cycles and time of the six GEMMs
# of one C2 step (ncu, serialised), the work the tail tiles remove independent of the clock
for t in 0 1; do
  PPMOE_TAIL128=$t timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.sum,sm__cycles_elapsed.avg.per_second --clock-control none --kernel-name-base demangled -k regex:grouped_gemm -c 12 --csv python tools/prof_step.py > gpurun_out/abt_$t.csv 2>&1
  python - $t <<PY
import csv, sys
t = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/abt_{t}.csv")) if len(r) > 14 and r[0].isdigit()]
by = {}
for r in rows:
    by.setdefault(int(r[0]), {"name": r[4]})[r[12]] = float(r[14].replace(",", ""))
ks = list(by.values())[-6:]
tot_c = sum(k["sm__pipe_tensor_cycles_active.sum"] for k in ks)
tot_t = sum(k["gpu__time_duration.sum"] for k in ks)
print(f"TAIL128={t}: tensor active {tot_c / 1e9:.4f} G cycles, time {tot_t / 1e6:.3f} ms; per GEMM (Mcyc):",
      [round(k["sm__pipe_tensor_cycles_active.sum"] / 1e6, 1) for k in ks])
PY
done
