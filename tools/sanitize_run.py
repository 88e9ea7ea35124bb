"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel family of the library on small inputs, including the
heavy-subtree sharing queue in its eager mode (hand-overs on a skewed graph),
the fused multi-motif query (prefix counting, sibling rows, resume), the
census, per-root counts, enumeration and a prefix-disconnected motif.  Counts
are checked against the oracle so a run that "passes" the sanitizer also
computed the right thing.
usage: compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2310_02800_b200 import motifs as M, synth, tmotif as T  # noqa: E402


def main():
    src, dst, t, n = synth.config_graph("C1", m=6000)
    og = oracle.Graph(src, dst, t, n)
    g = T.Graph(src, dst, t, n)
    mo = T.Motif(M.TRI, 3600)
    c = T.tm_count(g, mo)
    assert c == og.mine(M.TRI, 3600)["count"]
    rows, nt = T.tm_enumerate(g, mo, max(c, 1), canonical=True)
    assert nt == c
    specs = [(M.P3, [1800] * 2), (M.TRI, [1800] * 2), (M.C4, [1800] * 3), (M.DIA, [1800] * 4)]
    got = T.tm_count_multi(g, [T.Motif(mm, 3600, f) for mm, f in specs])
    assert got == [og.mine(mm, 3600, f)["count"] for mm, f in specs], got
    # again: the window descriptors now use the first-record ids the first query recorded
    assert T.tm_count_multi(g, [T.Motif(mm, 3600, f) for mm, f in specs]) == got
    assert list(T.tm_census36(g, 3600)) == [og.mine(M.P36[k], 3600)["count"] for k in range(36)]
    allr = np.arange(len(src), dtype=np.uint64)
    pr = T.tm_count_roots(g, T.Motif(M.C4, 3600), allr)
    assert np.array_equal(pr, og.mine(M.C4, 3600, roots=allr, per_root=True)["per_root"])
    dis = [(0, 1), (2, 3), (1, 2)]
    assert T.tm_count(g, T.Motif(dis, 3600)) == og.mine(dis, 3600)["count"]
    # skewed graph, sharing on (0) and eager (2): the inter-CTA hand-over queue
    s2, d2, t2, n2 = synth.burst_graph(231002806, m_bg=4000, core=32)
    og2 = oracle.Graph(s2, d2, t2, n2)
    g2 = T.Graph(s2, d2, t2, n2)
    shared = 0
    for share in (0, 2):
        for mm, f in ((M.C4, None), (M.TT, None), (M.DIA, [None, 900, None, 1800])):
            assert T.tm_count(g2, T.Motif(mm, 3600, f), share=share) == og2.mine(mm, 3600, f)["count"]
            shared += T.tm_last_run_info()["shared_tasks"]
    vl = (np.arange(n) % 2).astype(np.int32)
    g.set_labels(vl, None)
    og.set_labels(vl, None)
    cons = dict(vlabels={0: 1}, anti=[(1, 0, 0, 600)])
    assert T.tm_count(g, T.Motif(M.TRI, 3600, **cons)) == og.mine(M.TRI, 3600, **cons)["count"]
    print(f"sanitize workload ok (shared tasks {shared})")


if __name__ == "__main__":
    main()
