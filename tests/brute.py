"""Brute force for tiny graphs — the definition of PAPER.md §2.1 applied
literally, used to pin the oracle (and, transitively, the CUDA path).

Independent of both the oracle and the CUDA code: pure Python, no adjacency
structure, no binary search, no Algorithm 1 book-keeping.  It walks every
index-increasing L-tuple of the time-sorted edge list, pruned only by the
δ-span, and checks each predicate of the definition directly:

* temporal order ``e_1 < ... < e_L`` under the (t, input index) total order
  (P:169 with reading Q1),
* ``t_L - t_1 <= δ`` (inclusive),
* ``t_{i+1} - t_i <= δ_i`` (inclusive),
* an injective vertex map φ with φ(u_i)=src(e_i), φ(v_i)=dst(e_i),
* generalized query: required vertex / edge labels, and
  anti-edges ¬(u_j, v_j, δ_ij) attached to edge i — no graph edge
  φ(u_j) -> φ(v_j) other than the tuple's own (reading Q22) with
  t in [t_i, t_i + δ_ij], found by scanning the WHOLE edge list.
"""
from __future__ import annotations

INF = (1 << 63) - 1


def sort_order(t):
    """edge id -> input position, ids ranked by (t, input index) (reading Q1)."""
    return sorted(range(len(t)), key=lambda i: (int(t[i]), i))


def sorted_edges(src, dst, t):
    order = sort_order(t)
    return ([int(src[i]) for i in order], [int(dst[i]) for i in order], [int(t[i]) for i in order], order)


def verify_match(S, D, T, motif, delta, fine, tup, VL=None, EL=None, vlabels=None, elabels=None, anti=None):
    """The definition's predicates for one tuple of sorted edge ids.  VL: graph
    vertex labels, EL: edge labels by sorted id (None = all 0); vlabels:
    {motif vertex: label}, elabels: per motif edge label or None; anti:
    [(u, v, attach, window)]."""
    L = len(motif)
    if len(tup) != L:
        return False
    if any(not (tup[i] < tup[i + 1]) for i in range(L - 1)):
        return False
    if T[tup[-1]] - T[tup[0]] > delta:
        return False
    if fine is not None:
        for i in range(L - 1):
            f = INF if fine[i] is None else fine[i]
            if T[tup[i + 1]] - T[tup[i]] > f:
                return False
    phi = {}
    for (mu, mv), e in zip(motif, tup):
        for x, g in ((mu, S[e]), (mv, D[e])):
            if x in phi and phi[x] != g:
                return False
            phi[x] = g
    if len(set(phi.values())) != len(phi):
        return False
    for x, lab in (vlabels or {}).items():
        if ((VL[phi[x]] if VL is not None else 0)) != lab:
            return False
    for i, lab in enumerate(elabels or []):
        if lab is not None and (EL[tup[i]] if EL is not None else 0) != lab:
            return False
    for (u, v, a, w) in (anti or []):
        ta = T[tup[a]]
        for e in range(len(S)):
            if e not in tup and S[e] == phi[u] and D[e] == phi[v] and ta <= T[e] <= ta + w:
                return False
    return True


def brute(src, dst, t, motif, delta, fine=None, *, vlab=None, elab=None, vlabels=None, elabels=None, anti=None):
    """Sorted list of all matching tuples (sorted edge ids).  vlab: labels per
    graph vertex; elab: labels per input edge."""
    S, D, T, order = sorted_edges(src, dst, t)
    EL = None if elab is None else [int(elab[i]) for i in order]
    VL = None if vlab is None else [int(x) for x in vlab]
    m, L = len(S), len(motif)
    out = []

    def rec(tup):
        if len(tup) == L:
            if verify_match(S, D, T, motif, delta, fine, tup, VL, EL, vlabels, elabels, anti):
                out.append(tuple(tup))
            return
        start = tup[-1] + 1 if tup else 0
        for e in range(start, m):
            if tup and T[e] - T[tup[0]] > delta:
                break
            rec(tup + [e])

    rec([])
    return sorted(out)


def prefix_count(src, dst, t, motif, delta, fine=None):
    """Counts of every prefix motif M[:l], l = 1..L (the number of search-tree
    nodes with l matched edges)."""
    res = []
    for l in range(1, len(motif) + 1):
        f = None if fine is None else list(fine[: l - 1])
        res.append(len(brute(src, dst, t, motif[:l], delta, f)))
    return res
