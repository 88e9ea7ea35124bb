"""The smaller BASELINE.json configs, for ncu captures and timing:
C1 (1k vertices / 20k edges, TRI, δ = 1 h, count + enumerate) and C3
(wiki-talk-shaped, 7.8 M edges, C4 / TT / TT2 with δ = 1 day, enumeration to
a buffer sized by a prior count).  Prints one JSON line per query with the
library's CUDA-event times and rows/s.
usage: python tools/profile_configs.py [--reps 3]"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2310_02800_b200 import motifs as M  # noqa: E402
from paper_2310_02800_b200 import synth  # noqa: E402
from paper_2310_02800_b200 import tmotif as T  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()

for cfg, names, delta in (("C1", ["TRI"], 3600), ("C3", ["C4", "TT", "TT2"], 86400)):
    src, dst, t, n = synth.config_graph(cfg)
    g = T.Graph(src, dst, t, n)
    for name in names:
        mo = T.Motif(M.get(name), delta)
        cnt = T.tm_count(g, mo)
        cinfo = T.tm_last_run_info()
        L = len(M.get(name))
        buf = torch.empty((max(cnt, 1), L), dtype=torch.int32, device="cuda")
        best = None
        for _ in range(a.reps):
            rows, n_total = T.tm_enumerate(g, mo, cnt, buf=buf)
            info = T.tm_last_run_info()
            best = info if best is None or info["total_ms"] < best["total_ms"] else best
        assert n_total == cnt
        print(json.dumps({"config": cfg, "m": len(src), "motif": name, "delta_s": delta, "matches": cnt,
                          "count_total_ms": round(cinfo["total_ms"], 4),
                          "enum_total_ms": round(best["total_ms"], 4), "enum_mine_ms": round(best["mine_ms"], 4),
                          "rows_per_s": cnt / (best["total_ms"] / 1e3),
                          "enum_write_GBps": cnt * L * 4 / (best["total_ms"] / 1e3) / 1e9,
                          "root_edges_per_s_count": len(src) / (cinfo["total_ms"] / 1e3)}), flush=True)
