"""Independent pins for the oracle: closed forms and library routines that fix
the count without Algorithm 1 (SURVEY.md §8(c) "What pins each part").
None of these share logic with oracle/ or with the CUDA path.
"""
from __future__ import annotations

import bisect
from collections import defaultdict

import networkx as nx
from networkx.algorithms.isomorphism import DiGraphMatcher

from brute import sorted_edges


def static_time_ordered_count(src, dst, t, motif):
    """δ = ∞ pin: Σ over injective static embeddings φ of M into G (networkx
    subgraph monomorphisms, a library routine) of the number of increasing
    chains e_1 < ... < e_L with e_i an edge φ(u_i)→φ(v_i).  With δ = ∞ the
    temporal definition reduces to exactly this."""
    S, D, T, _ = sorted_edges(src, dst, t)
    pairs = defaultdict(list)
    G = nx.DiGraph()
    for e, (a, b) in enumerate(zip(S, D)):
        if a != b:
            pairs[(a, b)].append(e)
            G.add_edge(a, b)
    M = nx.DiGraph()
    M.add_edges_from(motif)
    total = 0
    for mapping in DiGraphMatcher(G, M).subgraph_monomorphisms_iter():
        phi = {mv: gv for gv, mv in mapping.items()}
        lists = [pairs[(phi[u], phi[v])] for (u, v) in motif]
        ways = [1] * len(lists[0])
        for i in range(1, len(lists)):
            prev, cur = lists[i - 1], lists[i]
            pref = [0]
            for w in ways:
                pref.append(pref[-1] + w)
            ways = [pref[bisect.bisect_left(prev, x)] for x in cur]
        total += sum(ways)
    return total


def two_node_closed_form(src, dst, t, delta):
    """Σ over the 4 two-node 3-edge motifs (0→1, x, y), x,y ∈ {0→1, 1→0}:
    every index-increasing triple of events on one vertex pair {a,b} with
    span <= δ is matched by exactly one of them, so the sum is
    Σ_pairs Σ_i C(n_i, 2), n_i = #{j > i on the pair : T_j - T_i <= δ}."""
    S, D, T, _ = sorted_edges(src, dst, t)
    byp = defaultdict(list)
    for e, (a, b) in enumerate(zip(S, D)):
        if a != b:
            byp[(min(a, b), max(a, b))].append(T[e])
    tot = 0
    for ts in byp.values():
        for i, ti in enumerate(ts):
            n_i = bisect.bisect_right(ts, ti + delta, lo=i + 1) - (i + 1)
            tot += n_i * (n_i - 1) // 2
    return tot


def census36_sum(src, dst, t, delta):
    """Σ over Paranjape's 36 motifs (0→1, E[a], E[b]) = number of
    index-increasing triples of the global edge list with span <= δ, no
    self-loop, and at most 3 distinct vertices (each such triple relabels by
    first appearance into exactly one of the 36).  No adjacency logic."""
    S, D, T, _ = sorted_edges(src, dst, t)
    m = len(S)
    tot = 0
    for i in range(m):
        if S[i] == D[i]:
            continue
        for j in range(i + 1, m):
            if T[j] - T[i] > delta:
                break
            if S[j] == D[j]:
                continue
            vj = {S[i], D[i], S[j], D[j]}
            if len(vj) > 3:
                continue
            for k in range(j + 1, m):
                if T[k] - T[i] > delta:
                    break
                if S[k] == D[k]:
                    continue
                if len(vj | {S[k], D[k]}) <= 3:
                    tot += 1
    return tot


def time_reverse(src, dst, t, motif, fine):
    """G^R: edge id i -> m-1-i with T' = C - T; M^R: motif edge order reversed,
    gaps reversed.  count(G, M, δ, δ_i) = count(G^R, M^R, δ, reversed δ_i)."""
    S, D, T, _ = sorted_edges(src, dst, t)
    C = max(T) if T else 0
    rs, rd, rt = S[::-1], D[::-1], [C - x for x in T[::-1]]
    rm = list(reversed(motif))
    rf = None if fine is None else list(reversed(fine))
    return rs, rd, rt, rm, rf
