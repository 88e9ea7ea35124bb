"""Host-side timing of the end-to-end step pieces exactly as bench.py's e2e
pass runs them (graph from pinned host memory, the fused query, graph close),
with the L2 flush and CUDA events of bench.py around the whole step."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2310_02800_b200 import synth  # noqa: E402
from paper_2310_02800_b200 import tmotif as T  # noqa: E402

src, dst, t, n = synth.config_graph(bench.CONFIG)
ph = [torch.from_numpy(x).pin_memory() for x in (src, dst, t)]
hs, hd, ht = (x.numpy() for x in ph)
s = torch.cuda.Stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
mos = [T.Motif(*bench.motif_fine(x)[:1], bench.DELTA, bench.motif_fine(x)[1]) for x in bench.MOTIFS]
for it in range(6):
    with torch.cuda.stream(s):
        flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    t0 = time.perf_counter()
    g = T.Graph(hs, hd, ht, n, stream=s)
    t1 = time.perf_counter()
    cs = T.tm_count_multi(g, mos, stream=s)
    t2 = time.perf_counter()
    g.close()
    t3 = time.perf_counter()
    e1.record(s)
    e1.synchronize()
    t4 = time.perf_counter()
    print(f"step {e0.elapsed_time(e1):.2f} ms (events)  create {1e3 * (t1 - t0):.1f}  query {1e3 * (t2 - t1):.1f}  "
          f"close {1e3 * (t3 - t2):.1f}  tail {1e3 * (t4 - t3):.1f} ms  {cs}", file=sys.stderr)
