#!/usr/bin/env python3
"""Per-launch table from an ncu --csv metrics log: one line per launch with
duration (us), DRAM MB, warp instructions (M) and issue activity."""
import csv, io, sys, collections
txt = [l for l in open(sys.argv[1]).read().splitlines() if l.startswith('"')]
rows = list(csv.reader(io.StringIO("\n".join(txt))))
h = rows[0]
ik, iid, im, iv = h.index("Kernel Name"), h.index("ID"), h.index("Metric Name"), h.index("Metric Value")
L = collections.OrderedDict()
for r in rows[1:]:
    d = L.setdefault(r[iid], {"k": r[ik].split("(")[0].split("::")[-1]})
    d[r[im]] = float(r[iv].replace(",", ""))
for i, d in L.items():
    print(f'{i:>4} {d["k"][:16]:16s} {d.get("gpu__time_duration.sum",0)/1e3:8.1f}us '
          f'{(d.get("dram__bytes_read.sum",0)+d.get("dram__bytes_write.sum",0))/1e6:8.1f}MB '
          f'{d.get("smsp__inst_executed.sum",0)/1e6:7.2f}Minst '
          f'issue {d.get("smsp__issue_active.avg.pct_of_peak_sustained_active",0):5.1f}%')
