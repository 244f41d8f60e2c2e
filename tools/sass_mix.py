"""Dynamic SASS opcode mix of one kernel from an ncu --set full report:
warp-instructions executed per opcode (and per matrix when --per N is given).
usage: python tools/sass_mix.py REPORT KERNEL_REGEX [--per N] [--top K]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
per = int(sys.argv[sys.argv.index("--per") + 1]) if "--per" in sys.argv else 0
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-name", "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = next(r for r in rows if r and r[0] == "Address")
ii, it, isrc = hdr.index("Instructions Executed"), hdr.index("Thread Instructions Executed"), hdr.index("Source")
ops, thr = collections.Counter(), collections.Counter()
tot = 0.0
for r in rows:
    if not r or not r[0].startswith("0x"):
        continue
    s = r[isrc].strip().split()
    if not s:
        continue
    op = s[1] if s[0].startswith("@") else s[0]
    op = op.rstrip(";")
    base = op.split(".")[0]
    if base == "IMAD" and ".MOV" in op:
        base = "IMAD.MOV"
    n = float(r[ii].replace(",", "") or 0)
    ops[base] += n
    thr[base] += float(r[it].replace(",", "") or 0)
    tot += n
print(f"total warp-instructions {tot:.4g}" + (f"  per matrix x32 (per-thread equiv) {tot / per * 32:.1f}" if per else ""))
for op, n in ops.most_common(top):
    pm = f" {n / per * 32:8.1f}/matrix" if per else ""
    print(f"{op:12s} {n / tot * 100:5.2f}%{pm}  lanes {thr[op] / max(n, 1):4.1f}")
