"""Prefix-fusion overhead probe: the 4-cycle alone (plain counting kernel)
against the 4-cycle carrying P3 (prefix-counting kernel), same query shape."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2310_02800_b200 import synth, tmotif as T  # noqa: E402
src, dst, t, n = synth.config_graph("C4")
g = T.Graph(src, dst, t, n)
mk = lambda x: T.Motif(*bench.motif_fine(x)[:1], bench.DELTA, bench.motif_fine(x)[1])  # noqa: E731
for label, ms in (("C4 alone", ["C4"]), ("P3 + C4", ["P3", "C4"]), ("DIA alone", ["DIA"]), ("TRI + DIA", ["TRI", "DIA"])):
    mos = [mk(x) for x in ms]
    best = None
    for _ in range(4):
        T.tm_count_multi(g, mos)
        k = max(x["mine_ms"] for x in T.tm_last_kernel_info())
        best = k if best is None else min(best, k)
    print(f"{label:10s} kernel {best:.3f} ms", file=sys.stderr)
