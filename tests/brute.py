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
* an injective vertex map φ with φ(u_i)=src(e_i), φ(v_i)=dst(e_i).
"""
from __future__ import annotations

INF = (1 << 63) - 1


def sort_order(t):
    """edge id -> input position, ids ranked by (t, input index) (reading Q1)."""
    return sorted(range(len(t)), key=lambda i: (int(t[i]), i))


def sorted_edges(src, dst, t):
    order = sort_order(t)
    return ([int(src[i]) for i in order], [int(dst[i]) for i in order], [int(t[i]) for i in order], order)


def verify_match(S, D, T, motif, delta, fine, tup):
    """The definition's predicates for one tuple of sorted edge ids."""
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
    return len(set(phi.values())) == len(phi)


def brute(src, dst, t, motif, delta, fine=None):
    """Sorted list of all matching tuples (sorted edge ids)."""
    S, D, T, _ = sorted_edges(src, dst, t)
    m, L = len(S), len(motif)
    out = []

    def rec(tup):
        if len(tup) == L:
            if verify_match(S, D, T, motif, delta, fine, tup):
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
