"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list into per-kernel shares.
    python tools/launch_summary.py launches.csv "header comment" > summary.csv"""
import collections
import csv
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")) if r]
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    k = r[ki][:60]
    n, t = agg.get(k, (0, 0.0))
    agg[k] = (n + 1, t + v)
tot = sum(t for _, t in agg.values())
if len(sys.argv) > 2:
    for line in sys.argv[2].split("\\n"):
        print("# " + line)
print("kernel,launches,total_ns,mean_ns,share")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k.replace(',', ';')},{n},{t:.0f},{t / n:.0f},{t / tot:.3f}")
