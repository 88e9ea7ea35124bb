import sys, torch; sys.path.insert(0,'/root/repo')
import bench
from paper_2310_02800_b200 import synth, tmotif as T
for m in (300_000, 2_000_000, 8_000_000, 20_000_000):
    src,dst,t,n = synth.config_graph("C4", m=m)
    g = T.Graph(src,dst,t,n)
    mk = lambda x: T.Motif(*bench.motif_fine(x)[:1], bench.DELTA, bench.motif_fine(x)[1])
    mos = [mk(x) for x in ["C4","TRI","DIA"]]
    print(m, "plain", T.tm_count_multi(g, mos, fuse=1), "fused", T.tm_count_multi(g, mos), flush=True)
