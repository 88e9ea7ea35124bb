"""One C5 query (TRI + 4-cycle, δ = 1 h, count, fused: TRI as the 4-cycle's
sibling rows) on one time slice of the 2e9-edge C5 graph, for ncu captures
and A/B timing of library variants (TMOTIF_LIB).
usage: python tools/c5_step.py [--parts 64] [--part 3] [--reps 3]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2310_02800_b200 import motifs as M, synth, tmotif as T  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--parts", type=int, default=64)
ap.add_argument("--part", type=int, default=3)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--no-pair", action="store_true", help="build the graph without the pair index")
ap.add_argument("--bucket-log2", type=int, default=0, help="tm_graph_opts.pair_id_bucket_log2")
a = ap.parse_args()
s, d, t, n, nr = synth.c5_rank_slice(a.part, a.parts, 3600)
g = T.Graph(s, d, t, n, pair_index=not a.no_pair, pair_id_bucket_log2=a.bucket_log2)
mos = [T.Motif(M.TRI, 3600), T.Motif(M.C4, 3600)]
best = None
for _ in range(a.reps):
    c = T.tm_count_multi(g, mos, root_range=(0, nr))
    info = T.tm_last_run_info()
    k = T.tm_last_kernel_info()
    if best is None or info["total_ms"] < best[0]["total_ms"]:
        best = (info, k, c)
info, k, c = best
print(json.dumps({"lib": T.LIB_PATH, "m": len(s), "roots": nr, "counts": c, "total_ms": info["total_ms"],
                  "horizon_ms": info["horizon_ms"], "mine_ms": [x["mine_ms"] for x in k],
                  "modes": [x["kernel_mode"] for x in k], "roots_per_s": 2 * nr / info["total_ms"] * 1e3}))
