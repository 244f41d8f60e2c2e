"""Summarise an ncu --set full report of one kernel by source line: top
instruction counts, divergent branches and lanes wasted (read here, after a
gpurun capture).  usage: python tools/ncu_lines.py REP KERNEL_REGEX [N]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
cur, hdr, res = None, None, []
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif r and r[0].isdigit() and hdr:
        def g(k):
            try:
                return float(r[hdr.index(k)].replace(",", ""))
            except (ValueError, IndexError):
                return 0.0
        res.append(dict(div=g("Divergent Branches"), ins=g("Instructions Executed"),
                        thr=g("Thread Instructions Executed"), smp=g("Warp Stall Sampling (All Samples)"),
                        f=cur, line=r[0], src=r[1][:100]))
tot = sum(x["ins"] for x in res)
tthr = sum(x["thr"] for x in res)
smp = sum(x["smp"] for x in res) or 1
print(f"warp-instr {tot:.0f}  lane util {tthr / tot / 32:.3f}")
byf = collections.Counter()
for x in res:
    byf[x["f"]] += x["ins"]
print({k: round(v / tot * 100, 1) for k, v in byf.most_common()})
print("-- divergent branches")
for x in sorted(res, key=lambda x: -x["div"])[:top]:
    if x["div"] == 0:
        break
    print(f"{x['div']:10.0f} {x['f']}:{x['line']} {x['src']}")
print("-- instructions / stall samples")
for x in sorted(res, key=lambda x: -x["ins"])[:top]:
    print(f"{x['ins'] / tot * 100:5.2f}% {x['smp'] / smp * 100:5.2f}% util {x['thr'] / max(x['ins'], 1) / 32:4.2f} "
          f"{x['f']}:{x['line']} {x['src']}")
print("-- idle lane-slots (instructions x inactive lanes)")
waste = sum(x["ins"] * 32 - x["thr"] for x in res)
for x in sorted(res, key=lambda x: -(x["ins"] * 32 - x["thr"]))[:top]:
    print(f"{(x['ins'] * 32 - x['thr']) / waste * 100:5.2f}% util {x['thr'] / max(x['ins'], 1) / 32:4.2f} "
          f"{x['f']}:{x['line']} {x['src']}")
