"""Key metrics of every kernel in an ncu report (duration, DRAM bytes,
instructions, occupancy, top stall reasons): python tools/ncu_summary.py REPORT"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h, units = r[0], r[1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__cycles_active.avg", "sm__inst_executed.avg.per_cycle_active"]
for row in r[2:]:
    print(row[h.index("Kernel Name")][:60])
    for k in keys:
        if k in h:
            print(f"   {k:55s} {row[h.index(k)]:>16} {units[h.index(k)]}")
    st = [(float(row[i] or 0), m) for i, m in enumerate(h)
          if m.startswith("smsp__pcsamp_warps_issue_stalled") and not m.endswith("not_issued")]
    tot = sum(v for v, _ in st) or 1
    for v, m in sorted(st, reverse=True)[:6]:
        print(f"   stall {m[33:]:45s} {v / tot:6.3f}")
