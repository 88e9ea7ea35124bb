"""Runs each bench query on the bench workload (for ncu captures and quick
A/B timing of library variants via TMOTIF_LIB).
usage: python tools/profile_queries.py [--config C4] [--motifs P3,TRI,C4,DIA] [--reps 1]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2310_02800_b200 import synth  # noqa: E402
from paper_2310_02800_b200 import tmotif as T  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default=bench.CONFIG)
ap.add_argument("--motifs", default=",".join(bench.MOTIFS))
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--grid", type=int, default=0, help="grid_ctas override")
a = ap.parse_args()
src, dst, t, n = synth.config_graph(a.config)
g = T.Graph(src, dst, t, n)
tot = 0.0
for name in a.motifs.split(","):
    mot, fine = bench.motif_fine(name)
    mo = T.Motif(mot, bench.DELTA, fine)
    best = None
    for _ in range(a.reps):
        c = T.tm_count(g, mo, grid_ctas=a.grid)
        info = T.tm_last_run_info()
        best = info if best is None or info["mine_ms"] < best["mine_ms"] else best
    tot += best["total_ms"]
    print(f"{name:5s} count={c} mine_ms={best['mine_ms']:.3f} horizon_ms={best['horizon_ms']:.3f} "
          f"grid={best['grid_ctas']}", file=sys.stderr)
print(f"sum total_ms={tot:.3f} lib={T.LIB_PATH}", file=sys.stderr)
