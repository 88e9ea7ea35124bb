"""Config C5 (BASELINE.json configs[4]: billion-edge power-law temporal graph,
time-range partitioned with δ-overlap halos across 8 × B200, TRI and C4,
δ = 1 h, counting) — one rank's share, on one GPU.

Rank `--rank` of `--world` draws only its slice (synth.c5_rank_slice: its
roots' time range plus the forward δ-halo), builds its graph and counts the
motifs over its roots exactly as bench.py's multi-GPU path does.  Parity:
per-root counts of every root in `--windows` random 10-minute windows of the
slice against the oracle (run on just the edges those roots can reach, which
by δ-locality, is all their matches need).
usage: python tools/c5_slice.py [--world 8] [--rank 0] [--reps 3] [--windows 6]"""
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
ap.add_argument("--world", type=int, default=8)
ap.add_argument("--rank", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--windows", type=int, default=6)
ap.add_argument("--motifs", default="TRI,C4")
ap.add_argument("--delta", type=int, default=3600)
a = ap.parse_args()

t0 = time.time()
src, dst, t, n, n_roots = synth.c5_rank_slice(a.rank, a.world, a.delta)
gen_s = time.time() - t0
m = len(src)
print(f"[c5] rank {a.rank}/{a.world}: m_slice={m} roots={n_roots} n={n} generated in {gen_s:.1f}s",
      file=sys.stderr, flush=True)
t0 = time.time()
g = T.Graph(src, dst, t, n)
build_s = time.time() - t0
res = {"workload": f"C5 billion-edge eth-shaped synthetic (BASELINE.json configs[4]), rank {a.rank} of {a.world}",
       "m_slice": m, "roots": n_roots, "n": n, "delta_s": a.delta, "generate_s": gen_s,
       "graph_build_s_incl_h2d": build_s, "motifs": []}
rng = np.random.default_rng(5)
for name in a.motifs.split(","):
    mo = T.Motif(M.get(name), a.delta)
    best = None
    for _ in range(a.reps):
        c = T.tm_count(g, mo, root_range=(0, n_roots))
        info = T.tm_last_run_info()
        if best is None or info["total_ms"] < best["total_ms"]:
            best = info
    # sampled per-root parity against the oracle
    import oracle
    checked = 0
    for _ in range(a.windows):
        w0 = int(rng.integers(0, max(1, n_roots - 1)))
        lo = w0
        hi = int(np.searchsorted(t, t[w0] + 600, side="left"))
        hi = min(max(hi, lo + 1), n_roots)
        reach = int(np.searchsorted(t, t[hi - 1] + a.delta, side="right"))
        og = oracle.Graph(src[lo:reach], dst[lo:reach], t[lo:reach], n)
        exp = og.mine(M.get(name), a.delta, roots=np.arange(hi - lo, dtype=np.uint64), per_root=True)["per_root"]
        got = T.tm_count_roots(g, mo, np.arange(lo, hi, dtype=np.uint64))
        assert np.array_equal(got, exp), (name, lo, hi)
        checked += hi - lo
    res["motifs"].append({"motif": name, "count": c, "total_ms": best["total_ms"], "mine_ms": best["mine_ms"],
                          "horizon_ms": best["horizon_ms"], "root_edges_per_s": n_roots / (best["total_ms"] / 1e3),
                          "matches_per_s": c / (best["total_ms"] / 1e3), "tail_ms": best["tail_ms"],
                          "warp_busy": best["warp_busy"], "parity_roots_checked": checked})
    print(f"[c5] {name}: count={c} total_ms={best['total_ms']:.2f} parity roots={checked}", file=sys.stderr, flush=True)
print(json.dumps(res))
