# Dev tool: fc1 forward GEMM under epilogue store / L2-hint variants -- time, DRAM bytes,
# tensor-pipe activity (ncu, one C2 step).  Measured: all four within 86.3-86.9 % tensor-active.
for v in "X=0" "PPMOE_STORE=cs" "PPMOE_STORE=v8" "PPMOE_HINT=1"; do
  env $v timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --kernel-name-base demangled -k regex:EpiFc1Fwd -c 2 --csv python tools/prof_step.py > gpurun_out/fc1_$v.csv 2>&1
  python - "$v" <<PY
import csv, sys
v = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/fc1_{v}.csv")) if len(r) > 14 and r[0].isdigit()]
by = {}
for r in rows:
    by.setdefault(int(r[0]), {})[r[12]] = float(r[14].replace(",", ""))
for k in list(by.values())[-1:]:
    print(v, {n.split(".")[0].split("__")[1]: round(x, 3) for n, x in k.items()})
PY
done
