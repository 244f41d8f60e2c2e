"""Per-stall-reason totals of a kernel's SASS, split at given address offsets (regions).
usage: python tools/stall_regions.py REPORT KERNEL_REGEX [OFFSET_HEX ...]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
cuts = sorted(int(x, 16) for x in sys.argv[3:])
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name", "regex:" + kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = next(r for r in rows if r and r[0] == "Address")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ii = hdr.index("Instructions Executed")
seen = set(); ex = []
for r in rows:
    if not r or not r[0].startswith("0x"): continue
    a = int(r[0], 16)
    if a in seen: continue
    seen.add(a); ex.append((a, r))
base = ex[0][0]
bounds = [0] + cuts + [1 << 60]
for lo, hi in zip(bounds, bounds[1:]):
    sel = [r for a, r in ex if lo <= a - base < hi]
    if not sel: continue
    tot = {k: sum(float(r[hdr.index(k)] or 0) for r in sel) for k in reasons}
    inst = sum(float(r[ii] or 0) for r in sel)
    s = sum(tot.values())
    print(f"[{lo:#x},{min(hi, ex[-1][0] - base):#x}) static {len(sel)} exec {inst:.3e} samples {int(s)}: " +
          ", ".join(f"{k[6:]}={int(v)}" for k, v in sorted(tot.items(), key=lambda kv: -kv[1]) if v > 0.01 * s))
