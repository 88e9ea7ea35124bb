"""Named motif catalog (inputs, not method arithmetic).

A motif is an ordered list of directed edges over motif vertices; list order
is the temporal order.  The paper's Fig. 6 (M1-M13) is lost
from PAPER.md, so these names follow SURVEY.md §8(d) and claim
no identity with the paper's M-numbers (reading Q19).
"""
from __future__ import annotations

TRI = [(0, 1), (1, 2), (2, 0)]                     # cyclic triangle (config C1)
P3 = [(0, 1), (1, 2), (2, 3)]                      # 3-path
C4 = [(0, 1), (1, 2), (2, 3), (3, 0)]              # temporal 4-cycle (reading Q20)
TT = [(0, 1), (1, 2), (2, 0), (0, 3)]              # tailed triangle
TT2 = [(0, 1), (1, 2), (2, 3), (3, 1)]             # tailed triangle, tail first
DIA = [(0, 1), (1, 2), (2, 0), (1, 3), (3, 2)]     # diamond, 5 edges
STAR3 = [(0, 1), (0, 2), (0, 3)]                   # out-star
PATH2 = [(0, 1), (1, 2)]

# Paranjape's 36 two/three-node three-edge motifs as (0→1, E[a], E[b]).
E6 = [(0, 1), (1, 0), (0, 2), (2, 0), (1, 2), (2, 1)]
P36 = [[(0, 1), E6[a], E6[b]] for a in range(6) for b in range(6)]
TWO_NODE = [mm for mm in P36 if max(max(e) for e in mm) == 1]   # the 4 two-node motifs

NAMED = {"TRI": TRI, "P3": P3, "C4": C4, "TT": TT, "TT2": TT2, "DIA": DIA, "STAR3": STAR3,
         "PATH2": PATH2}

# per-config motif sets (BASELINE.json configs)
CONFIG_MOTIFS = {
    "C1": ["TRI"],
    "C2": [f"P36_{a}{b}" for a in range(6) for b in range(6)],
    "C3": ["C4", "TT", "TT2"],
    "C4": ["P3", "TRI", "C4", "DIA"],
}


def get(name: str):
    if name.startswith("P36_"):
        a, b = int(name[4]), int(name[5])
        return P36[a * 6 + b]
    return NAMED[name]
