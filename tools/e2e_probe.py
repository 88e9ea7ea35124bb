"""Host-side timing of the end-to-end pieces (graph build from pinned host
memory, queries) on the bench workload."""
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
mos = [T.Motif(*bench.motif_fine(x)[:1], bench.DELTA, bench.motif_fine(x)[1]) for x in bench.MOTIFS]
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = T.Graph(hs, hd, ht, n, stream=s)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    for mo in mos:
        T.tm_count(g, mo, stream=s)
    t2 = time.perf_counter()
    g.close()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"build {1e3 * (t1 - t0):.1f} ms  queries {1e3 * (t2 - t1):.1f} ms  destroy {1e3 * (t3 - t2):.1f} ms",
          file=sys.stderr)

# the same through tm_count_multi, and a graph kept alive in between (as bench.py's timed part)
keep = T.Graph(hs, hd, ht, n, stream=s)
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = T.Graph(hs, hd, ht, n, stream=s)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    T.tm_count_multi(g, mos, stream=s)
    t2 = time.perf_counter()
    g.close()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"[multi, another graph resident] build {1e3 * (t1 - t0):.1f} ms  queries {1e3 * (t2 - t1):.1f} ms  "
          f"destroy {1e3 * (t3 - t2):.1f} ms", file=sys.stderr)
keep.close()
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = T.Graph(hs, hd, ht, n, stream=s)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    T.tm_count_multi(g, mos, stream=s)
    t2 = time.perf_counter()
    g.close()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"[multi] build {1e3 * (t1 - t0):.1f} ms  queries {1e3 * (t2 - t1):.1f} ms  destroy {1e3 * (t3 - t2):.1f} ms",
          file=sys.stderr)
