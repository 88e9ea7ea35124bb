import sys, torch; sys.path.insert(0,'/root/repo')
import bench
from paper_2310_02800_b200 import synth, tmotif as T
src,dst,t,n = synth.config_graph("C4")
g = T.Graph(src,dst,t,n)
mk = lambda x: T.Motif(*bench.motif_fine(x)[:1], bench.DELTA, bench.motif_fine(x)[1])
mos = [mk(x) for x in bench.MOTIFS]
print("plain", T.tm_count_multi(g, mos, fuse=1))
print("fused", T.tm_count_multi(g, mos)); print(T.tm_last_kernel_info())
print("fused rr", T.tm_count_multi(g, mos, root_range=(0, len(src))))
s = torch.cuda.Stream()
print("fused stream", T.tm_count_multi(g, mos, stream=s))
print("C4 TRI DIA", T.tm_count_multi(g, [mos[2], mos[1], mos[3]]))
print("TRI DIA", T.tm_count_multi(g, [mos[1], mos[3]]))
