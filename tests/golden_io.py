"""Reader for tests/golden/*.txt fixtures (each file carries its citation)."""
from __future__ import annotations

import glob
import os

INF = (1 << 63) - 1
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _groups(s):
    s = s.strip()
    if s == "-":
        return []
    return [[x for x in g.split()] for g in s.split("|")]


def load(path):
    d = {}
    for line in open(path):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        k, v = line.split(":", 1)
        d[k.strip()] = v.strip()
    edges = _groups(d["edges"])
    src = [int(e[0]) for e in edges]
    dst = [int(e[1]) for e in edges]
    t = [int(e[2]) for e in edges]
    motif = [(int(a), int(b)) for a, b in _groups(d["motif"])]
    delta = INF if d["delta"] == "inf" else int(d["delta"])
    fine = None
    if d["fine"] != "-":
        fine = [INF if x == "inf" else int(x) for x in d["fine"].split()]
    rows = sorted(tuple(int(x) for x in g) for g in _groups(d["rows"]))
    n = max(src + dst) + 1 if src else 1
    # generalized query (optional keys): anti: u v attach window | ...;
    # vlab: label per graph vertex; elab: label per input edge;
    # mvlabels: motif-vertex:label ...; melabels: per motif edge label or *
    anti = [tuple(int(x) for x in g) for g in _groups(d["anti"])] if "anti" in d else None
    vlab = [int(x) for x in d["vlab"].split()] if "vlab" in d else None
    elab = [int(x) for x in d["elab"].split()] if "elab" in d else None
    mvl = {int(a): int(b) for a, b in (x.split(":") for x in d["mvlabels"].split())} if "mvlabels" in d else None
    mel = [None if x == "*" else int(x) for x in d["melabels"].split()] if "melabels" in d else None
    return dict(name=os.path.basename(path), src=src, dst=dst, t=t, n=n, motif=motif, delta=delta,
                fine=fine, count=int(d["count"]), rows=rows, anti=anti, vlab=vlab, elab=elab, vlabels=mvl,
                elabels=mel)


def all_fixtures():
    return [load(p) for p in sorted(glob.glob(os.path.join(GOLDEN, "*.txt")))]
