"""Top stalled SASS instructions of a kernel in an ncu --set full report.
usage: python tools/stall_top.py REPORT KERNEL_REGEX [TOP]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name", "regex:" + kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = next(r for r in rows if r and r[0] == "Address")
ii, isrc, ism = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
ex = [(int(r[0], 16), float(r[ii] or 0), float(r[ism] or 0), r[isrc]) for r in rows if r and r[0].startswith("0x")]
seen = set(); ex2 = []
for e in ex:
    if e[0] in seen: continue
    seen.add(e[0]); ex2.append(e)
ex = ex2
base = ex[0][0]
tot = sum(e[2] for e in ex)
print("instrs", len(ex), "samples", int(tot), "warp-inst", int(sum(e[1] for e in ex)))
for a, n, sm, sx in sorted(ex, key=lambda e: -e[2])[:top]:
    print(f"{a - base:#7x} exec {int(n):9d} samples {int(sm):6d} {100 * sm / tot:5.1f}%  {sx.strip()[:90]}")
