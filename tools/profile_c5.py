"""One C5 time slice (rank 0 of 8), TRI and C4 counted once each — for ncu
captures of the C5 mining kernels.  usage: python tools/profile_c5.py [--no-stats]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2310_02800_b200 import motifs as M  # noqa: E402
from paper_2310_02800_b200 import synth  # noqa: E402
from paper_2310_02800_b200 import tmotif as T  # noqa: E402

stats = "--no-stats" not in sys.argv
src, dst, t, n, nr = synth.c5_rank_slice(3, 8, 3600)
g = T.Graph(src, dst, t, n)
for name in ("TRI", "C4"):
    c = T.tm_count(g, T.Motif(M.get(name), 3600), root_range=(0, nr))
    i = T.tm_last_run_info()
    print(name, c, i["mine_ms"], i["horizon_ms"], file=sys.stderr)
    if not stats:
        continue
    st = T.tm_search_stats_run(g, T.Motif(M.get(name), 3600), root_range=(0, nr))
    print(name, "nodes", st["nodes"][:4], "window_sum", st["window_sum"], "fast", st["fast_window_sum"], file=sys.stderr)
