"""Seeded test-case generators shared by the oracle pins and the GPU parity
tests (inputs only — no method arithmetic)."""
from __future__ import annotations

import random

from paper_2310_02800_b200 import motifs as M

INF = (1 << 63) - 1


def random_motif(rng: random.Random, L: int, max_v: int = 6):
    """Prefix-connected motif (every edge after the first touches an earlier
    vertex, reading Q9), vertex ids by first appearance."""
    edges = [(0, 1)]
    nv = 2
    for _ in range(L - 1):
        a = rng.randrange(nv)
        if nv < max_v and rng.random() < 0.5:
            b = nv
            nv += 1
        else:
            b = rng.randrange(nv - 1)
            if b >= a:
                b += 1
        edges.append((a, b) if rng.random() < 0.5 else (b, a))
    return edges


def reverse_prefix_connected(motif):
    seen = set(motif[-1])
    for u, v in reversed(motif[:-1]):
        if u not in seen and v not in seen:
            return False
        seen |= {u, v}
    return True


CATALOG = [M.TRI, M.P3, M.C4, M.TT, M.TT2, M.DIA, M.STAR3, M.PATH2, [(0, 1)], [(0, 1), (1, 0)],
           [(0, 1), (0, 1), (0, 1)], [(0, 1), (1, 0), (0, 1)]]


def random_fine(rng: random.Random, L: int):
    if L < 2 or rng.random() < 0.5:
        return None
    return [rng.choice([0, 1, 2, 4, 7, 15, INF]) for _ in range(L - 1)]
