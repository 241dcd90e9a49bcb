"""Hottest SASS lines (warp-stall samples) of one kernel in an ncu report:
python tools/ncu_sass_hot.py REPORT KERNEL_REGEX [N]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
r = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = r[0]
si, wi, ii = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
def num(v):
    try:
        return float(v or 0)
    except ValueError:
        return None


rows = [x for x in r[1:] if len(x) == len(h) and num(x[wi]) is not None]
tot = sum(float(x[wi] or 0) for x in rows)
ins = sum(float(x[ii] or 0) for x in rows)
print(f"samples {tot:.0f}  instructions {ins:.0f}")
for k, x in enumerate(rows):
    x.append(k)
for x in sorted(rows, key=lambda x: -float(x[wi] or 0))[:n]:
    print(f"{float(x[wi] or 0) / tot:6.3f} {x[ii]:>10} {x[-1]:5d} {x[si][:90]}")
