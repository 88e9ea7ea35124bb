"""Per-source-line warp-stall attribution: joins the SASS stall samples of an
.ncu-rep kernel with the -lineinfo line table of the same kernel's cubin.
usage: python tools/sass_lines.py REP KERNEL_REGEX OBJ_FILE MANGLED_SUBSTR [N] [SKIP] [COLUMN]
COLUMN: a source-page column, default "Warp Stall Sampling (All Samples)"; e.g.
"Instructions Executed" for where the warp instructions go."""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, kre, obj, msub = sys.argv[1:5]
obj = os.path.abspath(obj)
N = int(sys.argv[5]) if len(sys.argv) > 5 else 25
SKIP = sys.argv[6] if len(sys.argv) > 6 else "0"   # launches of KERNEL_REGEX to skip
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name-base", os.environ.get("NCU_NAME_BASE", "demangled"), "--kernel-name",
                      f"regex:{kre}", "--launch-skip", SKIP, "--launch-count", "1"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]
COL = sys.argv[7] if len(sys.argv) > 7 else "Warp Stall Sampling (All Samples)"
S = hdr.index(COL)
data = [r for r in rows[1:] if r and r[0].startswith("0x") and len(r) == len(hdr)]
base = int(data[0][0], 16)
samples = [(int(r[0], 16) - base, float((r[S] or "0").replace(",", "")), r[1].strip()) for r in data]
# line table
td = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", obj], cwd=td, capture_output=True)
cub = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
syms = subprocess.run(["cuobjdump", "-elf", os.path.join(td, cub)], capture_output=True, text=True).stdout
dis = subprocess.run(["nvdisasm", "-gi", os.path.join(td, cub)], capture_output=True, text=True).stdout
# find the function block
cur, fn_lines, line, fresh = None, {}, None, True
for l in dis.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", l)
    if m:
        cur = m.group(1)
        continue
    if cur is None or msub not in cur:
        continue
    m = re.search(r"//## File \"([^\"]+)\", line (\d+)(?: inlined at \"([^\"]+)\", line (\d+))?", l)
    if m:
        if fresh:   # innermost location of the next instruction (+ its call site)
            line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            if m.group(3):
                line += f" <- {m.group(4)}"
            fresh = False
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m:
        fresh = True
        if line:
            fn_lines[int(m.group(1), 16)] = line
agg = {}
tot = sum(s for _, s, _ in samples)
for off, s, ins in samples:
    ln = fn_lines.get(off, "?")
    agg[ln] = agg.get(ln, 0) + s
for ln, s in sorted(agg.items(), key=lambda kv: -kv[1])[:N]:
    print(f"{s / tot * 100:5.1f}%  {ln}")
