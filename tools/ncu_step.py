"""One bench-shaped query (tm_count_multi over the bench's motifs on config
C4) for `ncu --set full -k regex:mine_kernel`: the launches are the step's
mining kernels in launch order (the 4-cycle kernel that also counts P3 and
writes TRI's rows, then the diamond resuming from them).  The query runs
twice: the first records the graph's first-record ids (NextIdCache), the
second is the steady state bench.py times — capture it with --launch-skip."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2310_02800_b200 import synth, tmotif as T  # noqa: E402
src, dst, t, n = synth.config_graph("C4")
g = T.Graph(src, dst, t, n)
mos = [T.Motif(*bench.motif_fine(x)[:1], bench.DELTA, bench.motif_fine(x)[1]) for x in bench.MOTIFS]
for _ in range(2):
    print(dict(zip(bench.MOTIFS, T.tm_count_multi(g, mos))), T.tm_last_kernel_info(), file=sys.stderr)
