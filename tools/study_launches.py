"""Print tools/study_launches.sh's CSV as one line per launch. usage: python tools/study_launches.py CSV"""
import collections
import csv
import sys

rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
h = rows[0]
ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = collections.OrderedDict()
for r in rows[1:]:
    d.setdefault((int(r[iid]), r[ik]), {})[r[im]] = float(r[iv].replace(",", ""))
tot = 0.0
for (i, k), m in d.items():
    name = k.replace("void <unnamed>::", "").replace("<unnamed>::", "").split("(")[0]
    t = m["gpu__time_duration.sum"] / 1e3
    tot += t
    print(f"{i:3d} {name:32s} {t:8.1f} us  {m['smsp__inst_executed.sum'] / 1e6:7.1f} M inst  issue "
          f"{m['smsp__issue_active.avg.pct_of_peak_sustained_active']:5.1f}%  regs {m['launch__registers_per_thread']:.0f}")
print(f"total {tot:.1f} us")
