"""Query-time structure cost of the bench query (horizons + window
descriptors, tm_run_info.horizon_ms) on config C4, best of 6."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2310_02800_b200 import synth, tmotif as T  # noqa: E402
src, dst, t, n = synth.config_graph("C4")
g = T.Graph(src, dst, t, n)
mos = [T.Motif(*bench.motif_fine(x)[:1], bench.DELTA, bench.motif_fine(x)[1]) for x in bench.MOTIFS]
best = None
for _ in range(6):
    c = T.tm_count_multi(g, mos)
    h = T.tm_last_run_info()["horizon_ms"]
    best = h if best is None else min(best, h)
print(f"horizon+descriptor ms {best:.3f} counts {c}", file=sys.stderr)
