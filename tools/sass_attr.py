"""Attribute a kernel's executed SASS (ncu --set full report) to source call
sites: each instruction goes to the innermost inlined frame that lies in
FOCUS (default kog2_fast.cuh), using nvdisasm -gi line info of the cubin the
report was taken from.  Prints, per focus line, warp-instructions per matrix
(x32 / COUNT), its share, IMAD.MOV / FP64 / int shares and average lanes.
usage: python tools/sass_attr.py REPORT KERNEL_REGEX OBJ COUNT [FOCUS] [TOP]"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, kern, obj, count = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
focus = sys.argv[5] if len(sys.argv) > 5 else "kog2_fast.cuh"
top = int(sys.argv[6]) if len(sys.argv) > 6 else 40
depth = int(os.environ.get("DEPTH", "1"))
# DISASM_KERNEL: regex on the mangled name when KERNEL_REGEX (demangled, for ncu) matches several cubin functions  # 2: attribute to the caller of the innermost focus frame
# FUNCS=1: attribute to the enclosing function (kernel or noinline callee) instead of a source line
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-name", "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = next(r for r in rows if r and r[0] == "Address")
ii, it, isrc = hdr.index("Instructions Executed"), hdr.index("Thread Instructions Executed"), hdr.index("Source")
ex = [(int(r[0], 16), float(r[ii] or 0), float(r[it] or 0), r[isrc].strip()) for r in rows if r and r[0].startswith("0x")]
base = ex[0][0]
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
kname = None
for cub in sorted(f for f in os.listdir(d) if f.endswith(".cubin")):  # the cubin that holds the kernel
    dis = subprocess.run(["nvdisasm", "-gi", os.path.join(d, cub)], capture_output=True, text=True).stdout.splitlines()
    for ln in dis:
        m = re.match(r"^(\S+):$", ln)
        if m and re.search(os.environ.get("DISASM_KERNEL", kern), m.group(1)) and not ln.startswith("."):
            kname = m.group(1)
            break
    if kname:
        break
start = dis.index(kname + ":")
func = kname
site = {}
chain = []
last_addr_line = False
for ln in dis[start + 1:]:
    if ln.startswith(".text."):  # the kernel's section ends (it holds its noinline callees too)
        break
    m = re.match(r"^(\S+):$", ln)
    if m and not ln.startswith(".L"):  # a callee's entry label
        func = m.group(1)
        continue
    m = re.match(r"\s*//## File \"([^\"]+)\", line (\d+)(?: inlined at \"([^\"]+)\", line (\d+))?", ln)
    if m:
        if last_addr_line:
            chain = []
            last_addr_line = False
        chain.append((os.path.basename(m.group(1)), int(m.group(2))))
        continue
    m = re.match(r"\s*/\*([0-9a-f]+)\*/", ln)
    if m:
        last_addr_line = True
        fr = [f"{f}:{l}" for f, l in chain if f == focus]
        s = fr[min(depth, len(fr)) - 1] if fr else (chain[-1][0] + ":" + str(chain[-1][1]) if chain else "?")
        site[int(m.group(1), 16)] = ("fn " + func.split("$")[-1][-60:]) if os.environ.get("FUNCS") else s
agg = collections.defaultdict(lambda: collections.Counter())
tot = 0.0
for a, n, t, src in ex:
    s = site.get(a - base, "?")
    op = src.split()[1] if src.startswith("@") else (src.split()[0] if src else "")
    if os.environ.get("OPC") and not op.startswith(os.environ["OPC"]):  # OPC=DSETP: one opcode family only
        continue
    c = agg[s]
    c["n"] += n
    c["t"] += t
    if op.startswith("IMAD.MOV") or op.startswith("MOV"):
        c["mov"] += n
    if op[:4] in ("DFMA", "DADD", "DMUL") or op.startswith("MUFU"):
        c["fp64"] += n
    tot += n
print(f"total {tot / count * 32:.1f} warp-instr per 32 matrices")
src_lines = {}
fp = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2407_13116_b200", "csrc", focus)
if os.path.exists(fp):
    src_lines = {i + 1: l.strip() for i, l in enumerate(open(fp))}
key = os.environ.get("SORT", "n")  # n | mov | fp64
for s, c in sorted(agg.items(), key=lambda kv: -kv[1][key])[:top]:
    ln = int(s.split(":")[1]) if s.startswith(focus) else 0
    print(f"{c['n'] / count * 32:7.1f} {c['n'] / tot * 100:5.1f}%  mov {c['mov'] / max(c['n'], 1) * 100:3.0f}%  fp64 "
          f"{c['fp64'] / max(c['n'], 1) * 100:3.0f}%  lanes {c['t'] / max(c['n'], 1):4.1f}  {s:22s} {src_lines.get(ln, '')[:70]}")
