import os, sys, time, torch
sys.path.insert(0, '/root/repo')
from paper_2310_02800_b200 import synth
from paper_2310_02800_b200 import tmotif as T
src, dst, t, n = synth.config_graph("C4")
ph = [torch.from_numpy(x).pin_memory() for x in (src, dst, t)]
hs, hd, ht = (x.numpy() for x in ph)
s = torch.cuda.Stream()
dsrc, ddst, dt = (torch.from_numpy(x.astype(x.dtype)).cuda() for x in (src.astype('int32'), dst.astype('int32'), t))
for it in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    g = T.Graph(hs, hd, ht, n, stream=s); torch.cuda.synchronize(); t1 = time.perf_counter(); g.close()
    g = T.Graph(dsrc, ddst, dt, n, stream=s); torch.cuda.synchronize(); t2 = time.perf_counter(); g.close()
    print(f"build from pinned host {1e3*(t1-t0):.1f} ms, from device {1e3*(t2-t1):.1f} ms", file=sys.stderr)
