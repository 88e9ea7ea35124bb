"""Top SASS instructions of one kernel in an .ncu-rep by warp-stall samples.
usage: python tools/ncu_hotspots.py REP KERNEL_REGEX [N]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name-base", "demangled", "--kernel-name",
                      f"regex:{kre}", "--launch-count", "1"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]
S = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
data = [r for r in rows[1:] if r and r[0] != "Address" and len(r) == len(hdr) and r[0].startswith("0x")]
tot = sum(float(r[S] or 0) for r in data)
agg = {}
for r in data:
    for i in stall_cols:
        agg[hdr[i]] = agg.get(hdr[i], 0) + float(r[i] or 0)
print(f"total stall samples {tot:.0f}")
print("  ".join(f"{k[6:]}={v / tot * 100:.1f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:10]))
data.sort(key=lambda r: -float(r[S] or 0))
for r in data[:N]:
    top = sorted(((float(r[i] or 0), hdr[i][6:]) for i in stall_cols), reverse=True)[:3]
    print(f"{float(r[S]) / tot * 100:5.1f}%  {r[0][-5:]}  {r[1].strip()[:60]:60s} " +
          " ".join(f"{n}:{v:.0f}" for v, n in top if v > 0))
