"""Per-kernel share of a `ncu --metrics gpu__time_duration.sum --csv` launch list.
usage: python tools/launch_summary.py LAUNCHES.csv"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[-3] == "gpu__time_duration.sum"]
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows:
    unit = r[-2]
    v = float(r[-1].replace(",", "")) * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0,
                                         "msecond": 1.0}.get(unit, 1e-6)
    name = r[4].split("(")[0]
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:45s} launches={cnt[k]:4d} total_ms={v:11.2f} mean_ms={v / cnt[k]:10.3f} share={v / T * 100:5.1f}%")
