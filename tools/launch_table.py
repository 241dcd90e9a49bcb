"""Per-kernel table of an ncu --csv launch list (gpu__time_duration.sum and,
when captured, dram__bytes_read/write.sum): python tools/launch_table.py CSV"""
import collections
import csv
import sys

r = list(csv.reader(open(sys.argv[1])))
hi = [i for i, x in enumerate(r) if "Kernel Name" in x][0]
h = r[hi]
rows = r[hi + 1:]
ki, mi, ni, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name"), h.index("ID")
agg = collections.defaultdict(lambda: collections.defaultdict(float))
ids = collections.defaultdict(set)
for x in rows:
    if len(x) <= mi:
        continue
    try:
        v = float(x[mi].replace(",", ""))
    except ValueError:
        continue
    k = x[ki][:60]
    agg[k][x[ni]] += v
    ids[k].add(x[ii])
tot = sum(a.get("gpu__time_duration.sum", 0) for a in agg.values())
print(f"{'kernel':60s} {'n':>4s} {'us/launch':>10s} {'share':>6s} {'DRAM GB/launch':>15s}")
for k, a in sorted(agg.items(), key=lambda t: -t[1].get("gpu__time_duration.sum", 0))[:22]:
    n = len(ids[k])
    t = a.get("gpu__time_duration.sum", 0)
    db = (a.get("dram__bytes_read.sum", 0) + a.get("dram__bytes_write.sum", 0)) / n / 1e9
    print(f"{k:60s} {n:4d} {t / n / 1e3:10.1f} {t / tot:6.3f} {db:15.3f}")
print(f"total {tot / 1e3:.1f} us")
