# Dev tool: fc1 forward GEMM with the paired vs scalar GeLU epilogue, interleaved rebuilds (ncu, one box).
for v in paired scalar paired scalar; do
  if [ $v = scalar ]; then make -B -j16 EXTRA=-DPPMOE_GELU_SCALAR > /dev/null 2>&1; else make -B -j16 > /dev/null 2>&1; fi
  timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum --clock-control none --kernel-name-base demangled -k regex:"EpiFc1Fwd" -c 2 --csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-a2a > gpurun_out/gab_$v.csv 2>&1
  python - $v <<PY
import csv, sys
v = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/gab_{v}.csv")) if len(r) > 14 and r[0].isdigit()]
by = {}
for r in rows:
    by.setdefault(int(r[0]), {})[r[12]] = float(r[14].replace(",", ""))
for k in by.values():
    print(v, {n.split(".")[0].split("__")[1]: round(x, 3) for n, x in k.items()})
PY
done
