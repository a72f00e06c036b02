"""Dev tool: summarise an ncu launch list (gpu__time_duration + dram bytes, --csv) of
`bench.py --steps 2`: per kernel of the LAST step, time, DRAM bytes and fraction of the
measured HBM peak.  usage: python tools/launch_summary.py launches.csv [peak_GBps]"""
import csv
import sys
from collections import OrderedDict

path = sys.argv[1]
peak = float(sys.argv[2]) if len(sys.argv) > 2 else 6528.7
rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[0].isdigit()]
by = OrderedDict()
for r in rows:
    by.setdefault(int(r[0]), {"name": r[4]})[r[12]] = float(r[14].replace(",", ""))
ks = list(by.values())
starts = [i for i, k in enumerate(ks) if "router_tc_prep" in k["name"] or "router_dmma" in k["name"]]
last = ks[starts[-2]:starts[-1]] if len(starts) >= 2 else ks
tot = sum(k.get("gpu__time_duration.sum", 0) for k in last)
print(f"{len(last)} launches in the last full step, {tot / 1e6:.3f} ms serialised (cold)")
for k in last:
    t = k.get("gpu__time_duration.sum", 0)
    b = k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0)
    nm = k["name"].split("(")[0].replace("void ", "").replace("ppmoe::", "")[:60]
    print(f"  {nm:60s} {t / 1e3:9.1f} us {b / 1e6:9.1f} MB  {b / t / peak if t else 0:5.2f} of HBM")
