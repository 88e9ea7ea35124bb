import sys; sys.path.insert(0, '/root/repo')
import bench
from paper_2310_02800_b200 import synth, motifs as M, tmotif as T
src, dst, t, n = synth.config_graph("C3")
g = T.Graph(src, dst, t, n)
mos = [T.Motif(*bench.motif_fine(x)[:1], bench.DELTA, bench.motif_fine(x)[1]) for x in bench.MOTIFS]
T.tm_count_multi(g, mos); print(T.tm_last_kernel_info())
for mo in mos:
    T.tm_count(g, mo); print(T.tm_last_run_info()["grid_ctas"])
