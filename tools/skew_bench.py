"""A/B of heavy-subtree sharing (tm_run_opts.share, §8 a8) on skewed graphs:
the bench workload (C4) and a burst workload (a C3-shaped background plus
dense cores whose few roots own most of the search work).
usage: python tools/skew_bench.py [--reps 3] [--core 256] [--bursts 4] [--hubs 4] [--fan 100000]
Prints one JSON line per (workload, motif, share) with the best mining time."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2310_02800_b200 import motifs as M  # noqa: E402
from paper_2310_02800_b200 import synth  # noqa: E402
from paper_2310_02800_b200 import tmotif as T  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--core", type=int, default=256)
ap.add_argument("--bursts", type=int, default=4)
ap.add_argument("--skip-c4", action="store_true")
ap.add_argument("--skip-cores", action="store_true")
ap.add_argument("--hubs", type=int, default=4)
ap.add_argument("--fan", type=int, default=100000)
a = ap.parse_args()


def run(tag, g, motifs):
    for name, delta, fine in motifs:
        mo = T.Motif(M.get(name), delta, fine)
        res = {}
        for share in (1, 0):
            best = None
            for _ in range(a.reps):
                c = T.tm_count(g, mo, share=share)
                info = T.tm_last_run_info()
                if best is None or info["mine_ms"] < best["mine_ms"]:
                    best = info
            res[share] = (c, best)
        assert res[0][0] == res[1][0]
        print(json.dumps({"workload": tag, "motif": name, "count": res[0][0],
                          "mine_ms_off": round(res[1][1]["mine_ms"], 3), "mine_ms_on": round(res[0][1]["mine_ms"], 3),
                          "shared_tasks": res[0][1]["shared_tasks"], "grid": res[0][1]["grid_ctas"],
                          "tail_ms_off": round(res[1][1]["tail_ms"], 3), "tail_ms_on": round(res[0][1]["tail_ms"], 3),
                          "warp_busy_off": round(res[1][1]["warp_busy"], 3),
                          "warp_busy_on": round(res[0][1]["warp_busy"], 3)}), flush=True)


if not a.skip_c4:
    src, dst, t, n = synth.config_graph("C4")
    g = T.Graph(src, dst, t, n)
    run("C4 bench workload", g, [(nm, bench.DELTA, [bench.FINE] * (len(M.get(nm)) - 1)) for nm in bench.MOTIFS])
    del g

def c3_plus(extra):
    src, dst, t, n = synth.config_graph("C3")
    parts = [(src, dst, t)] + extra(n, int(t.max()))
    return (np.concatenate([p[0] for p in parts]).astype(np.uint32),
            np.concatenate([p[1] for p in parts]).astype(np.uint32),
            np.concatenate([p[2] for p in parts]).astype(np.int64), n)


def cores(n, span):
    """dense cores: every ordered pair of `core` vertices once within 1 h"""
    rng = np.random.default_rng(7)
    out = []
    for _ in range(a.bursts):
        vs = rng.choice(n, a.core, replace=False)
        x, y = np.meshgrid(vs, vs, indexing="ij")
        k = x != y
        t0 = int(rng.integers(0, span - 3600))
        out.append((x[k], y[k], t0 + rng.integers(0, 3600, int(k.sum()))))
    return out


def fans(n, span):
    """fan bursts: a hub gets 4 edges (the heavy roots), then sends `fan`
    edges to distinct vertices within 12 h, each of which sends 8 edges within
    the next 6 h — a handful of search trees with ~fan*8 nodes each"""
    rng = np.random.default_rng(11)
    out = []
    for _ in range(a.hubs):
        h = int(rng.integers(0, n))
        t0 = int(rng.integers(0, span - 86400))
        xs = rng.choice(n, 4, replace=False)
        out.append((xs, np.full(4, h), t0 + np.arange(4)))
        ys = rng.choice(n, a.fan, replace=False)
        ty = t0 + 4 + np.sort(rng.integers(0, 43200, a.fan))
        out.append((np.full(a.fan, h), ys, ty))
        zs = rng.integers(0, n, 8 * a.fan)
        out.append((np.repeat(ys, 8), zs, np.repeat(ty, 8) + rng.integers(0, 21600, 8 * a.fan)))
    return out


if not a.skip_cores:
    src, dst, t, n = c3_plus(cores)
    g = T.Graph(src, dst, t, n)
    tag = f"C3 + {a.bursts} dense {a.core}-vertex cores (m={len(src)})"
    run(tag, g, [("TRI", 86400, None), ("P3", 86400, None), ("C4", 86400, [3600, 3600, 3600]), ("TT", 86400, None)])
    del g
src, dst, t, n = c3_plus(fans)
g = T.Graph(src, dst, t, n)
tag = f"C3 + {a.hubs} fan bursts of {a.fan} (m={len(src)})"
run(tag, g, [("P3", 86400, None), ("C4", 86400, None), ("TT", 86400, None)])
