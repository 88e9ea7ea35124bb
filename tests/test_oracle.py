"""Pins for the oracle (oracle/tmoracle.c, Algorithm 1) against things other
than itself: the paper's worked rules, the literal definition (brute force),
closed forms, a library routine (networkx monomorphisms) at δ = ∞, and
symmetries/invariants of the definition."""
from __future__ import annotations

import random

import numpy as np
import pytest

import oracle
from brute import brute, prefix_count, sorted_edges, verify_match
from cases import CATALOG, INF, random_fine, random_motif, reverse_prefix_connected
from golden_io import all_fixtures
from paper_2310_02800_b200 import motifs as M
from paper_2310_02800_b200 import synth
from pins import census36_sum, static_time_ordered_count, time_reverse, two_node_closed_form


def ocount(src, dst, t, n, motif, delta, fine=None):
    return oracle.Graph(src, dst, t, n).mine(motif, delta, fine)["count"]


def orows(src, dst, t, n, motif, delta, fine=None):
    r = oracle.Graph(src, dst, t, n).mine(motif, delta, fine, enumerate_=True)
    return sorted(tuple(int(x) for x in row) for row in r["rows"]), r["n_total"]


# --------------------------------------------------------------- worked examples
def fx_cons(fx):
    return dict(vlabels=fx["vlabels"], elabels=fx["elabels"], anti=fx["anti"])


@pytest.mark.parametrize("fx", all_fixtures(), ids=lambda f: f["name"])
def test_golden(fx):
    og = oracle.Graph(fx["src"], fx["dst"], fx["t"], fx["n"])
    if fx["vlab"] is not None or fx["elab"] is not None:
        og.set_labels(fx["vlab"], fx["elab"])
    r = og.mine(fx["motif"], fx["delta"], fx["fine"], enumerate_=True, **fx_cons(fx))
    rows = sorted(tuple(int(x) for x in row) for row in r["rows"])
    assert r["n_total"] == fx["count"]
    assert rows == fx["rows"]
    # the fixture itself is consistent with the literal definition
    assert brute(fx["src"], fx["dst"], fx["t"], fx["motif"], fx["delta"], fx["fine"], vlab=fx["vlab"],
                 elab=fx["elab"], **fx_cons(fx)) == fx["rows"]


# ------------------------------------------------------------------ brute force
def _trials(n_trials, seed0, L_choices, m_range, tmax=30):
    rng = random.Random(seed0)
    for k in range(n_trials):
        L = rng.choice(L_choices)
        motif = rng.choice([c for c in CATALOG if len(c) == L] + [random_motif(rng, L)])
        m = rng.randint(*m_range)
        n = rng.randint(3, 9)
        src, dst, t, n = synth.tiny_graph(seed0 * 1000 + k, n=n, m=m, tmax=tmax)
        delta = rng.choice([0, 3, 10, 25, INF])
        fine = random_fine(rng, L)
        yield src, dst, t, n, motif, delta, fine


@pytest.mark.parametrize("seed", range(6))
def test_oracle_vs_brute_L123(seed):
    for src, dst, t, n, motif, delta, fine in _trials(40, 100 + seed, [1, 2, 3], (0, 70)):
        rows, n_total = orows(src, dst, t, n, motif, delta, fine)
        b = brute(src, dst, t, motif, delta, fine)
        assert rows == b, (motif, delta, fine)
        assert n_total == len(b) == ocount(src, dst, t, n, motif, delta, fine)


@pytest.mark.parametrize("seed", range(4))
def test_oracle_vs_brute_L45(seed):
    for src, dst, t, n, motif, delta, fine in _trials(20, 200 + seed, [4, 5], (5, 36), tmax=40):
        if delta == INF and len(motif) == 5:
            delta = 25
        rows, n_total = orows(src, dst, t, n, motif, delta, fine)
        assert rows == brute(src, dst, t, motif, delta, fine), (motif, delta, fine)


def test_search_nodes_equal_prefix_counts():
    """nodes[l] (partial matches with l edges whose next window is searched) is
    the count of the l-edge prefix motif; every window is searched once."""
    for src, dst, t, n, motif, delta, fine in _trials(30, 7, [2, 3, 4], (5, 40)):
        st = oracle.Graph(src, dst, t, n).mine(motif, delta, fine)["stats"]
        pc = prefix_count(src, dst, t, motif, delta, fine)
        assert st["nodes"][1:len(motif)] == pc[:-1]
        assert st["matches"] == pc[-1]


def test_window_sum_single_list_motifs():
    """Σ|window| for motifs whose every level has one bound endpoint (no list
    choice): windows are the bound vertex's out/in edges after e_l within δ
    and δ_l, counted here from brute-force prefix matches."""
    rng = random.Random(11)
    for k in range(30):
        motif = rng.choice([M.P3, M.STAR3, M.PATH2, [(0, 1), (2, 1), (3, 2)]])
        src, dst, t, n = synth.tiny_graph(500 + k, n=6, m=rng.randint(5, 45), tmax=30)
        delta = rng.choice([0, 5, 12, INF])
        fine = random_fine(rng, len(motif))
        S, D, T, _ = sorted_edges(src, dst, t)
        exp = 0
        for l in range(1, len(motif)):
            fl = None if fine is None else fine[:l - 1]
            for tup in brute(src, dst, t, motif[:l], delta, fl):
                phi = {}
                for (a, b), e in zip(motif[:l], tup):
                    phi[a], phi[b] = S[e], D[e]
                u, v = motif[l]
                f = INF if fine is None or fine[l - 1] is None else fine[l - 1]
                for c in range(tup[-1] + 1, len(S)):
                    ok_list = (S[c] == phi[u]) if u in phi else (D[c] == phi[v])
                    if ok_list and T[c] - T[tup[0]] <= delta and T[c] - T[tup[-1]] <= f:
                        exp += 1
        st = oracle.Graph(src, dst, t, n).mine(motif, delta, fine)["stats"]
        assert st["window_sum"] == exp


def test_instrumentation_both_mapped_levels_shorter_list():
    """Pins the oracle's list choice for a motif edge with both endpoints
    mapped ("N_out(u_G)/N_in(v_G)", reading Q8: the shorter list by
    degree, a tie takes N_in(v_G)): window_sum, list_sum and probe_sum are
    recomputed here from brute-force prefix matches and per-vertex degrees
    counted off the global edge list.  Choosing the other list (or always
    one of them) changes these counters but not the matches."""
    rng = random.Random(12)
    motifs = [M.TRI, M.C4, M.DIA, M.TT, [(0, 1), (1, 0), (0, 1)], [(0, 1), (1, 2), (0, 2)],
              [(0, 1), (1, 2), (2, 1), (1, 0)]]
    for k in range(40):
        motif = motifs[k % len(motifs)]
        src, dst, t, n = synth.tiny_graph(1500 + k, n=rng.randint(3, 6), m=rng.randint(8, 40 if len(motif) < 5 else 28),
                                          tmax=rng.choice([12, 30]))
        delta = rng.choice([5, 12, INF] if len(motif) < 5 else [5, 12])
        fine = random_fine(rng, len(motif))
        S, D, T, _ = sorted_edges(src, dst, t)
        m = len(S)
        out_deg = [sum(1 for c in range(m) if S[c] == x) for x in range(n)]
        in_deg = [sum(1 for c in range(m) if D[c] == x) for x in range(n)]
        win = lst = probes = 0
        for l in range(1, len(motif)):
            fl = None if fine is None else fine[:l - 1]
            for tup in brute(src, dst, t, motif[:l], delta, fl):
                phi = {}
                for (a, b), e in zip(motif[:l], tup):
                    phi[a], phi[b] = S[e], D[e]
                u, v = motif[l]
                if u in phi and v in phi:
                    use_out = out_deg[phi[u]] < in_deg[phi[v]]
                else:
                    use_out = u in phi
                x = phi[u] if use_out else phi[v]
                length = out_deg[x] if use_out else in_deg[x]
                lst += length
                probes += length.bit_length()      # ceil(log2(len + 1))
                f = INF if fine is None or fine[l - 1] is None else fine[l - 1]
                for c in range(tup[-1] + 1, m):
                    on_list = (S[c] == x) if use_out else (D[c] == x)
                    if on_list and T[c] - T[tup[0]] <= delta and T[c] - T[tup[-1]] <= f:
                        win += 1
        st = oracle.Graph(src, dst, t, n).mine(motif, delta, fine)["stats"]
        assert (st["window_sum"], st["list_sum"], st["probe_sum"]) == (win, lst, probes), (motif, delta, fine)


# ----------------------------------------------------------------- closed forms
def test_delta_inf_equals_static_time_ordered_count():
    rng = random.Random(5)
    for k in range(40):
        L = rng.choice([2, 3, 4])
        motif = rng.choice([c for c in CATALOG if len(c) == L] + [random_motif(rng, L, max_v=4)])
        src, dst, t, n = synth.tiny_graph(900 + k, n=rng.randint(3, 7), m=rng.randint(4, 30), tmax=12)
        assert ocount(src, dst, t, n, motif, INF) == static_time_ordered_count(src, dst, t, motif), motif


def test_two_node_closed_form():
    for k in range(30):
        src, dst, t, n = synth.tiny_graph(1300 + k, n=4, m=60, tmax=40)
        for delta in (0, 4, 13, INF):
            s = sum(ocount(src, dst, t, n, mm, delta) for mm in M.TWO_NODE)
            assert s == two_node_closed_form(src, dst, t, delta)


def test_census36_sum():
    for k in range(12):
        src, dst, t, n = synth.tiny_graph(1700 + k, n=5, m=50, tmax=40)
        for delta in (0, 6, 20):
            s = sum(ocount(src, dst, t, n, mm, delta) for mm in M.P36)
            assert s == census36_sum(src, dst, t, delta)


def test_single_edge_motif_counts_non_self_loops():
    src, dst, t, n = synth.tiny_graph(3, n=5, m=200, tmax=50, p_self=0.2)
    assert ocount(src, dst, t, n, [(0, 1)], 0) == int(np.sum(src != dst))


# ---------------------------------------------------------- symmetries/invariants
def test_delta_monotone_and_fine_subsumption():
    rng = random.Random(9)
    for k in range(15):
        motif = rng.choice(CATALOG[:6])
        src, dst, t, n = synth.tiny_graph(2000 + k, n=6, m=60, tmax=50)
        g = oracle.Graph(src, dst, t, n)
        prev = -1
        for d in (0, 1, 3, 7, 15, 30, 60, INF):
            c = g.mine(motif, d)["count"]
            assert c >= prev
            prev = c
            L = len(motif)
            # every δ_i >= δ: equal to the coarse-only count
            assert g.mine(motif, d, [d] * (L - 1))["count"] == c
            # lowering one δ_i never increases the count
            f = [INF] * (L - 1)
            f[rng.randrange(L - 1)] = 2
            assert g.mine(motif, d, f)["count"] <= c


def test_time_reversal_direction_reversal_shift_relabel():
    rng = random.Random(13)
    for k in range(30):
        motif = rng.choice([c for c in CATALOG if len(c) >= 2 and reverse_prefix_connected(c)])
        L = len(motif)
        src, dst, t, n = synth.tiny_graph(2500 + k, n=6, m=50, tmax=40)
        delta = rng.choice([3, 10, 25, INF])
        fine = random_fine(rng, L)
        base = ocount(src, dst, t, n, motif, delta, fine)
        rs, rd, rt, rm, rf = time_reverse(src, dst, t, motif, fine)
        assert ocount(rs, rd, rt, n, rm, delta, rf) == base
        assert ocount(dst, src, t, n, [(b, a) for a, b in motif], delta, fine) == base
        assert ocount(src, dst, np.asarray(t) + 10**12, n, motif, delta, fine) == base
        perm = np.random.default_rng(k).permutation(n).astype(np.uint32)
        assert ocount(perm[src], perm[dst], t, n, motif, delta, fine) == base
        sh = np.random.default_rng(k + 1).permutation(len(src))
        assert ocount(src[sh], dst[sh], t[sh], n, motif, delta, fine) == base or \
            _ties_reordered(t, sh)


def _ties_reordered(t, sh):
    # shuffling input changes the (t, input index) tie order among equal
    # timestamps, which can legitimately change counts (reading Q1); only
    # accept a difference when equal timestamps exist.
    return len(set(t.tolist())) < len(t)


def test_input_order_independence_unique_times():
    rng = np.random.default_rng(1)
    for k in range(10):
        m = 60
        src, dst, _, n = synth.tiny_graph(3000 + k, n=6, m=m)
        t = rng.permutation(200)[:m].astype(np.int64)  # unique timestamps
        base = ocount(src, dst, t, n, M.TRI, 40)
        sh = rng.permutation(m)
        assert ocount(src[sh], dst[sh], t[sh], n, M.TRI, 40) == base


def test_concatenation_sums():
    a = synth.tiny_graph(41, n=6, m=50, tmax=30)
    b = synth.tiny_graph(42, n=6, m=50, tmax=30)
    for motif in (M.TRI, M.C4, M.PATH2):
        ca = ocount(*a, motif, 10)
        cb = ocount(*b, motif, 10)
        src = np.concatenate([a[0], b[0]]); dst = np.concatenate([a[1], b[1]])
        t = np.concatenate([a[2], b[2] + 1000])
        assert ocount(src, dst, t, 6, motif, 10) == ca + cb


def test_partition_halo_sums():
    """A match belongs to the partition holding e_1 (reading Q16); mining each
    root range [lo,hi) on the edge slice [lo, H_δ(hi-1)] sums to the total
    (P:1025-1037)."""
    rng = random.Random(17)
    for k in range(20):
        motif = rng.choice(CATALOG)
        src, dst, t, n = synth.tiny_graph(3500 + k, n=7, m=80, tmax=60)
        delta = rng.choice([0, 5, 15])
        S, D, T, _ = sorted_edges(src, dst, t)
        S, D, T = np.array(S, np.uint32), np.array(D, np.uint32), np.array(T, np.int64)
        total = ocount(S, D, T, n, motif, delta)
        cuts = sorted(rng.sample(range(1, 80), 3))
        bounds = [0] + cuts + [80]
        s = 0
        for lo, hi in zip(bounds[:-1], bounds[1:]):
            ehi = int(np.searchsorted(T, T[hi - 1] + delta, side="right"))  # one past H_δ(hi-1)
            g = oracle.Graph(S[lo:ehi], D[lo:ehi], T[lo:ehi], n)
            s += g.mine(motif, delta, root_range=(0, hi - lo))["count"]
        assert s == total


def test_per_root_and_enumeration_consistency():
    src, dst, t, n = synth.tiny_graph(77, n=6, m=120, tmax=60)
    g = oracle.Graph(src, dst, t, n)
    for motif in (M.TRI, M.TT, M.C4):
        r = g.mine(motif, 20, per_root=True)
        e = g.mine(motif, 20, enumerate_=True)
        assert int(r["per_root"].sum()) == r["count"] == e["n_total"]
        S, D, T, _ = sorted_edges(src, dst, t)
        rows = [tuple(int(x) for x in row) for row in e["rows"]]
        assert len(set(rows)) == len(rows)
        assert all(verify_match(S, D, T, motif, 20, None, row) for row in rows)
        roots = np.bincount([row[0] for row in rows], minlength=len(S))
        assert np.array_equal(roots, r["per_root"].astype(np.int64))


def test_truncated_enumeration_keeps_exact_total():
    src, dst, t, n = synth.tiny_graph(78, n=5, m=100, tmax=40)
    g = oracle.Graph(src, dst, t, n)
    full = g.mine(M.TRI, 20)["count"]
    assert full > 5
    e = g.mine(M.TRI, 20, enumerate_=True, cap=5)
    assert e["n_total"] == full and len(e["rows"]) == 5


def test_multithreaded_equals_single():
    src, dst, t, n = synth.config_graph("C1")
    g = oracle.Graph(src, dst, t, n)
    a = g.mine(M.TRI, 3600, threads=1)
    b = g.mine(M.TRI, 3600, threads=4)
    assert a["count"] == b["count"] and a["stats"] == b["stats"]


def test_validation():
    g = oracle.Graph(np.array([0], np.uint32), np.array([1], np.uint32), np.array([0], np.int64), 2)
    assert g.mine([(0, 1), (2, 3)], 5)["count"] == 0   # prefix-disconnected: AllEdges (Q9)
    with pytest.raises(oracle.OracleError):
        g.mine([(0, 0)], 5)                  # motif self-loop
    with pytest.raises(oracle.OracleError):
        g.mine([(0, 1)], -1)                 # δ < 0
    with pytest.raises(oracle.OracleError):
        oracle.Graph(np.array([0], np.uint32), np.array([5], np.uint32), np.array([0], np.int64), 2)
    e = oracle.Graph(np.zeros(0, np.uint32), np.zeros(0, np.uint32), np.zeros(0, np.int64), 3)
    assert e.mine(M.TRI, 10)["count"] == 0   # empty graph is valid


def test_c5_slices_agree_and_tile():
    """The C5 time-slice generator (input infrastructure): overlapping slices
    agree on their shared events, adjacent rank slices tile the roots, and
    each rank's halo is exactly the next rank's first δ-window."""
    from paper_2310_02800_b200 import synth
    import dataclasses
    spec = dataclasses.replace(synth.C5, m=20_000_000, span=synth.C5.span)   # same shape, 1 % of the events
    day = 86400
    a = synth.c5_slice(5 * day, 8 * day, spec=spec)
    b = synth.c5_slice(6 * day, 9 * day, spec=spec)
    lo, hi = 6 * day + spec.t0, 8 * day + spec.t0
    ka, kb = (a[2] >= lo), (b[2] < hi)
    assert ka.sum() > 1000
    for x, y in zip(a[:3], b[:3]):
        assert np.array_equal(x[ka], y[kb])
    assert np.all(np.diff(a[2]) >= 0)
    w = 4000
    r0 = synth.c5_rank_slice(0, w, 3600, spec=spec)
    r1 = synth.c5_rank_slice(1, w, 3600, spec=spec)
    n0 = r0[4]
    halo = r0[2][n0:]
    tb = spec.span // w + spec.t0                   # the rank boundary
    assert np.all(r0[2][:n0] < tb) and np.all(r1[2] >= tb)
    assert len(halo) == np.searchsorted(r1[2], tb + 3600, "right")   # exactly the next δ-window
    assert np.array_equal(r0[0][n0:], r1[0][:len(halo)])



# ------------------------------------------- generalized query: labels, anti-edges
def random_constraints(rng, motif, n_labels):
    """Random label requirements and anti-edges over the motif's vertices."""
    verts = sorted({x for e in motif for x in e})
    vl = {v: rng.randrange(n_labels) for v in verts if rng.random() < 0.3} or None
    el = [rng.randrange(n_labels) if rng.random() < 0.25 else None for _ in motif]
    el = el if any(x is not None for x in el) else None
    anti = []
    for _ in range(rng.choice([0, 0, 1, 1, 2])):
        u, v = rng.sample(verts, 2)
        anti.append((u, v, rng.randrange(len(motif)), rng.choice([0, 2, 5, 12, 40])))
    return vl, el, anti or None


@pytest.mark.parametrize("seed", range(6))
def test_labels_and_anti_edges_vs_brute(seed):
    """Oracle = the literal definition (brute force scanning the whole edge list
    for anti-edge witnesses) on random small multigraphs with duplicate
    timestamps, labels and up to two anti-edges per motif."""
    rng = random.Random(4200 + seed)
    for k in range(40):
        n = rng.randint(2, 7)
        src, dst, t, _ = synth.tiny_graph(seed * 1000 + k, n=n, m=rng.randint(0, 45), tmax=rng.randint(4, 40))
        L = rng.choice([1, 2, 3, 3, 4])
        motif = rng.choice([c for c in CATALOG if len(c) == L] + [random_motif(rng, L)])
        nl = rng.choice([1, 2, 3])
        vlab = [rng.randrange(nl) for _ in range(n)] if rng.random() < 0.7 else None
        elab = [rng.randrange(nl) for _ in range(len(src))] if rng.random() < 0.5 else None
        vl, el, anti = random_constraints(rng, motif, nl)
        delta = rng.choice([0, 3, 10, 25, INF])
        fine = random_fine(rng, L)
        og = oracle.Graph(src, dst, t, n)
        if vlab is not None or elab is not None:
            og.set_labels(vlab, elab)
        r = og.mine(motif, delta, fine, enumerate_=True, vlabels=vl, elabels=el, anti=anti)
        got = sorted(tuple(int(x) for x in row) for row in r["rows"])
        exp = brute(src, dst, t, motif, delta, fine, vlab=vlab, elab=elab, vlabels=vl, elabels=el, anti=anti)
        assert got == exp, (seed, k, motif, delta, fine, vl, el, anti)


def test_constraint_invariants():
    """Invariants the definition implies: requirements can only remove matches;
    an always-satisfied label requirement changes nothing; an anti-edge with a
    pair the graph never has changes nothing; widening an anti window never
    adds matches; all-distinct labels split the count exactly."""
    src, dst, t, n = synth.tiny_graph(77, n=6, m=120, tmax=80)
    og = oracle.Graph(src, dst, t, n)
    base = og.mine(M.TRI, 30)["count"]
    assert base > 0
    og.set_labels([0] * n, [0] * len(src))
    assert og.mine(M.TRI, 30, vlabels={0: 0, 1: 0, 2: 0}, elabels=[0, 0, 0])["count"] == base
    # labels 0/1 per vertex: the counts over the 2^3 label assignments of the motif vertices sum to base
    lab = [v % 2 for v in range(n)]
    og.set_labels(lab, None)
    tot = sum(og.mine(M.TRI, 30, vlabels={0: a, 1: b, 2: c})["count"] for a in (0, 1) for b in (0, 1) for c in (0, 1))
    assert tot == base
    # edge labels by input position parity, per motif edge: sums over assignments again
    og.set_labels(None, [i % 2 for i in range(len(src))])
    tot = sum(og.mine(M.TRI, 30, elabels=[a, b, c])["count"] for a in (0, 1) for b in (0, 1) for c in (0, 1))
    assert tot == base
    # anti-edges: monotone in the window, bounded by the unconstrained count
    prev = base
    for w in (0, 1, 3, 10, 30, 100):
        c = og.mine(M.TRI, 30, anti=[(0, 2, 0, w)])["count"]
        assert c <= prev
        prev = c
    # a vertex the graph never touches as a target: the anti pair never exists
    src2 = np.concatenate([src, [n]]).astype(np.uint32)
    dst2 = np.concatenate([dst, [0]]).astype(np.uint32)
    t2 = np.concatenate([t, [10**6]]).astype(np.int64)
    og2 = oracle.Graph(src2, dst2, t2, n + 1)
    assert og2.mine(M.TRI, 30)["count"] == base
    with pytest.raises(oracle.OracleError):
        og.mine(M.TRI, 30, anti=[(0, 0, 0, 5)])
    with pytest.raises(oracle.OracleError):
        og.mine(M.TRI, 30, anti=[(0, 7, 0, 5)])
    with pytest.raises(oracle.OracleError):
        og.mine(M.TRI, 30, anti=[(0, 1, 3, 5)])


# ------------------------------------------------ prefix-disconnected motifs (Q9)
DISCONNECTED = [[(0, 1), (2, 3)], [(0, 1), (2, 3), (1, 2)], [(0, 1), (2, 3), (3, 0)],
                [(0, 1), (2, 3), (4, 5)], [(0, 1), (1, 2), (3, 4), (4, 0)], [(0, 1), (2, 1), (3, 4)]]


@pytest.mark.parametrize("seed", range(3))
def test_disconnected_motifs_vs_brute(seed):
    """A motif edge that touches no earlier motif vertex takes its candidates
    from all later edges (Alg. 1's AllEdges branch)."""
    rng = random.Random(900 + seed)
    for k in range(24):
        motif = DISCONNECTED[k % len(DISCONNECTED)]
        src, dst, t, n = synth.tiny_graph(seed * 100 + k, n=rng.randint(4, 9), m=rng.randint(0, 40), tmax=30)
        delta = rng.choice([0, 3, 10, INF])
        fine = random_fine(rng, len(motif))
        rows, n_total = orows(src, dst, t, n, motif, delta, fine)
        assert rows == brute(src, dst, t, motif, delta, fine), (motif, delta, fine)


def test_disjoint_edge_pairs_closed_form():
    """[(0,1), (2,3)] with δ = ∞ counts the vertex-disjoint pairs of non-loop
    edges: C(m,2) − Σ_v C(d_v,2) + Σ_{a<b} C(c_ab,2) by inclusion–exclusion
    (d_v = edges at v, c_ab = edges between a and b in either direction)."""
    from math import comb
    for seed in range(6):
        src, dst, t, n = synth.tiny_graph(4000 + seed, n=12, m=150, tmax=1000)
        keep = src != dst
        src, dst, t = src[keep], dst[keep], t[keep]
        deg = np.bincount(np.concatenate([src, dst]), minlength=n)
        pairs = {}
        for a, b in zip(src.tolist(), dst.tolist()):
            key = (min(a, b), max(a, b))
            pairs[key] = pairs.get(key, 0) + 1
        want = comb(len(src), 2) - sum(comb(int(d), 2) for d in deg) + sum(comb(c, 2) for c in pairs.values())
        assert ocount(src, dst, t, n, [(0, 1), (2, 3)], INF) == want
