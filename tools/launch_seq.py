"""Print the kernel sequence between the last two launches of a marker kernel
in an ncu --metrics gpu__time_duration.sum csv (one query batch)."""
import csv
import io
import sys

path, marker = sys.argv[1], sys.argv[2]
txt = open(path).read()
lines = [ln for ln in txt.splitlines() if ln.startswith('"')]
r = [x for x in csv.DictReader(io.StringIO("\n".join(lines)))
     if x["Metric Name"] == "gpu__time_duration.sum"]
idx = [i for i, x in enumerate(r) if marker in x["Kernel Name"]]
s, e = idx[-2], idx[-1]
tot = 0.0
for x in r[s:e]:
    v = float(x["Metric Value"].replace(",", ""))
    u = x["Metric Unit"]
    v = v / 1000 if u == "ns" else v * 1000 if u == "ms" else v
    tot += v
    print(f"{v:9.1f} {x['Grid Size']:>14} {x['Block Size']:>12} {x['Kernel Name'][:80]}")
print(f"total {tot:.1f} us")
