import os, sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2310_02800_b200 import synth, motifs as M, tmotif as T
z = "/tmp/tm_ab_C4.npz"
if os.path.exists(z):
    d = np.load(z); src, dst, t, n = d["src"], d["dst"], d["t"], int(d["n"])
else:
    src, dst, t, n = synth.config_graph("C4")
g = T.Graph(src, dst, t, n)
spec = [("P3", [21600] * 2), ("TRI", [21600] * 2), ("C4", [21600] * 3), ("DIA", [21600] * 4)]
mos = [T.Motif(M.get(nm), 86400, f) for nm, f in spec]
lo = int(sys.argv[1]) if len(sys.argv) > 1 else 0
w = int(sys.argv[2]) if len(sys.argv) > 2 else 2000000
print(T.tm_count_multi(g, mos, root_range=(lo, lo + w)), flush=True)
