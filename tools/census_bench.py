"""Config C2 (BASELINE.json configs[1]: email-Eu-core-shaped, all 36
Paranjape motifs, δ = 1 h, counting): the fused census (tm_census36, one
traversal) against 36 separate tm_count queries, best of --reps, CUDA-event
times inside the library (horizons + mining).  Prints one JSON line.
usage: python tools/census_bench.py [--reps 5]"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2310_02800_b200 import motifs as M  # noqa: E402
from paper_2310_02800_b200 import synth  # noqa: E402
from paper_2310_02800_b200 import tmotif as T  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
src, dst, t, n = synth.config_graph("C2")
g = T.Graph(src, dst, t, n)
mos = [T.Motif(M.P36[k], 3600) for k in range(36)]
best_sep, best_fused, sep_counts, fused = None, None, None, None
for _ in range(a.reps):
    tot, hz, mine, cs = 0.0, 0.0, 0.0, []
    for mo in mos:
        cs.append(T.tm_count(g, mo))
        i = T.tm_last_run_info()
        tot += i["total_ms"]
        hz += i["horizon_ms"]
        mine += i["mine_ms"]
    if best_sep is None or tot < best_sep[0]:
        best_sep = (tot, hz, mine)
    sep_counts = cs
    fused = T.tm_census36(g, 3600)
    i = T.tm_last_run_info()
    if best_fused is None or i["total_ms"] < best_fused[0]:
        best_fused = (i["total_ms"], i["horizon_ms"], i["mine_ms"])
assert np.array_equal(fused, np.array(sep_counts, np.uint64))
m = len(src)
print(json.dumps({"workload": "C2 email-Eu-core-shaped synthetic (BASELINE.json configs[1])", "m": m, "n": n,
                  "delta_s": 3600, "motifs": 36, "matches": int(fused.sum()),
                  "separate_36_queries": {"total_ms": best_sep[0], "horizon_ms": best_sep[1], "mine_ms": best_sep[2]},
                  "fused_census": {"total_ms": best_fused[0], "horizon_ms": best_fused[1], "mine_ms": best_fused[2]},
                  "speedup": best_sep[0] / best_fused[0],
                  "root_edges_per_s_fused": 36 * m / (best_fused[0] / 1000),
                  "matches_per_s_fused": float(fused.sum()) / (best_fused[0] / 1000)}))
