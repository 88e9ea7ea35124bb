"""Locality probe: the bench query (P3/TRI/C4/DIA on C4) over P time slices
of the graph, each its own resident graph (roots + forward δ-halo, the
multi-GPU split of multi.rank_slice) mined one after the other on one GPU.
Each slice's lists then span 1/P of the time axis, so the query's random
record reads stay within a P-times smaller region; the sum of the slices'
mining times against the whole-graph kernel measures what that locality is
worth (the slices pay their own launches and tails).
usage: python tools/slice_probe.py [P ...]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2310_02800_b200 import multi, synth, tmotif as T  # noqa: E402

Ps = [int(x) for x in sys.argv[1:]] or [1, 4, 16]
cache = "/tmp/tm_ab_C4.npz"
if os.path.exists(cache):
    z = np.load(cache)
    src, dst, t, n = z["src"], z["dst"], z["t"], int(z["n"])
else:
    src, dst, t, n = synth.config_graph("C4")
names = bench.MOTIFS
mos = [T.Motif(*bench.motif_fine(x)[:1], bench.DELTA, bench.motif_fine(x)[1]) for x in names]
reach = max(multi.reach(bench.DELTA, bench.motif_fine(x)[1]) for x in names)
stream = torch.cuda.Stream()
for P in Ps:
    tot, mine, counts = 0.0, 0.0, np.zeros(len(names), np.int64)
    for r in range(P):
        lo, hi, eh = multi.rank_slice(t, reach, P, r)
        g = T.Graph(src[lo:eh], dst[lo:eh], t[lo:eh], n, device=0, stream=stream)
        T.tm_count_multi(g, mos, root_range=(0, hi - lo), stream=stream)   # records the first-record ids
        best = None
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            c = T.tm_count_multi(g, mos, root_range=(0, hi - lo), stream=stream)
            e1.record(stream)
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            mm = sum(x["mine_ms"] for x in T.tm_last_kernel_info())
            if best is None or ms < best[0]:
                best = (ms, mm, c)
        tot += best[0]
        mine += best[1]
        counts += np.asarray(best[2], np.int64)
        g.close()
    print(json.dumps({"P": P, "step_ms_sum": round(tot, 3), "mine_ms_sum": round(mine, 3),
                      "counts": dict(zip(names, [int(x) for x in counts]))}), flush=True)
