"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv):
per-kernel total time and share over the last `steps` of the run.
usage: launch_summary.py file.csv [steps_total] [steps_keep]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
total_steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
keep = int(sys.argv[3]) if len(sys.argv) > 3 else 1
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            data.append(d)
per = len(data) // total_steps
step = data[per * (total_steps - keep):]
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
tot = collections.OrderedDict()
for d in step:
    k = d["Kernel Name"].split("(")[0][:70]
    v = float(d["Metric Value"].replace(",", "")) * scale[d["Metric Unit"]]
    tot.setdefault(k, [0.0, 0])
    tot[k][0] += v
    tot[k][1] += 1
s = sum(v[0] for v in tot.values())
print(f"{'us':>10} {'n':>4} {'share':>6}  kernel   (last {keep} of {total_steps} steps)")
for k, v in sorted(tot.items(), key=lambda x: -x[1][0]):
    print(f"{v[0]:10.1f} {v[1]:4d} {100 * v[0] / s:5.1f}%  {k}")
print(f"{s:10.1f} us total per {keep} step(s)")
