"""Runtime specialisation (tm_motif_specialise, NVRTC) against the generic
kernel, on the C4 bench workload: a motif outside the build-time catalog and
Table-5-style constrained 4-cycle queries (V, V+T, V+T+A) on random vertex
labels.  Best of --reps mining times (CUDA events in the library) and the
one-off compile time.  Prints one JSON line per query.
usage: python tools/rtc_bench.py [--reps 3]"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2310_02800_b200 import motifs as M  # noqa: E402
from paper_2310_02800_b200 import synth  # noqa: E402
from paper_2310_02800_b200 import tmotif as T  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
src, dst, t, n = synth.config_graph("C4")
g = T.Graph(src, dst, t, n)
g.set_labels(np.random.default_rng(3).integers(0, 2, n).astype(np.int32), None)
day, six = 86400, 21600
queries = [("C4 + chord 0->3 (not in the catalog)", [(0, 1), (1, 2), (2, 3), (0, 3)], day, [six] * 3, {}),
           ("C4, V (labels)", M.C4, day, None, {"vlabels": {0: 0, 2: 1}}),
           ("C4, V+T", M.C4, day, [six] * 3, {"vlabels": {0: 0, 2: 1}}),
           ("C4, V+T+A (anti 2->0 on edge 2, P:632)", M.C4, day, [six] * 3,
            {"vlabels": {0: 0, 2: 1}, "anti": [(2, 0, 2, 3600)]})]


def best(mo):
    b, c = None, None
    for _ in range(a.reps):
        c = T.tm_count(g, mo)
        i = T.tm_last_run_info()
        b = i if b is None or i["mine_ms"] < b["mine_ms"] else b
    return c, b


for name, mot, d, f, cons in queries:
    c0, i0 = best(T.Motif(mot, d, f, **cons))
    mo = T.Motif(mot, d, f, **cons)
    t0 = time.perf_counter()
    mo.specialise()
    comp = time.perf_counter() - t0
    c1, i1 = best(mo)
    assert c0 == c1
    print(json.dumps({"query": name, "count": c1, "generic_mine_ms": round(i0["mine_ms"], 3),
                      "specialised_mine_ms": round(i1["mine_ms"], 3), "speedup": i0["mine_ms"] / i1["mine_ms"],
                      "compile_s": round(comp, 2), "roots": len(src),
                      "root_edges_per_s": len(src) / (i1["total_ms"] / 1e3)}), flush=True)
