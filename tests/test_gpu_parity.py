"""Parity of the CUDA path (through the C ABI) with the oracle, element by
element on the same seeded inputs.  Everything here is integer work, so the
bar is bit-exact: counts, per-root counts, canonical-sorted enumerations and
the search-tree instrumentation counters."""
from __future__ import annotations

import random

import numpy as np
import pytest

import oracle
from brute import brute, sorted_edges, verify_match
from cases import CATALOG, INF, random_fine, random_motif, reverse_prefix_connected
from golden_io import all_fixtures
from paper_2310_02800_b200 import motifs as M
from paper_2310_02800_b200 import synth
from paper_2310_02800_b200 import tmotif as T
from pins import census36_sum, time_reverse, two_node_closed_form

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    T.lib()


def gpu_rows(g, mo, cap=None):
    if cap is None:
        cap = T.tm_count(g, mo)
    rows, n_total = T.tm_enumerate(g, mo, cap, canonical=True)
    return [tuple(int(x) for x in r) for r in rows], n_total


def check_case(src, dst, t, n, motif, delta, fine, *, rows=True, stats=True, roots=True):
    og = oracle.Graph(src, dst, t, n)
    exp = og.mine(motif, delta, fine, enumerate_=rows)
    g = T.Graph(src, dst, t, n)
    mo = T.Motif(motif, delta, fine)
    c = T.tm_count(g, mo)
    assert c == exp["count"], (motif, delta, fine)
    if rows:
        r, n_total = gpu_rows(g, mo)
        assert n_total == exp["n_total"]
        assert r == [tuple(int(x) for x in row) for row in exp["rows"]]
    if stats:
        st = T.tm_search_stats_run(g, mo)
        os_ = exp["stats"]
        assert st["nodes"][:len(motif)] == os_["nodes"][:len(motif)]
        assert (st["window_sum"], st["list_sum"], st["probe_sum"], st["matches"]) == \
            (os_["window_sum"], os_["list_sum"], os_["probe_sum"], os_["matches"])
    if roots and len(src):
        allr = np.arange(len(src), dtype=np.uint64)
        pr = og.mine(motif, delta, fine, roots=allr, per_root=True)["per_root"]
        assert np.array_equal(T.tm_count_roots(g, mo, allr), pr)
    return c


# ------------------------------------------------------------ worked examples
@pytest.mark.parametrize("fx", all_fixtures(), ids=lambda f: f["name"])
def test_golden(fx):
    g = T.Graph(np.array(fx["src"]), np.array(fx["dst"]), np.array(fx["t"]), fx["n"])
    if fx["vlab"] is not None or fx["elab"] is not None:
        g.set_labels(fx["vlab"], fx["elab"])
    mo = T.Motif(fx["motif"], fx["delta"], fx["fine"], vlabels=fx["vlabels"], elabels=fx["elabels"],
                 anti=fx["anti"])
    assert T.tm_count(g, mo) == fx["count"]
    r, n_total = gpu_rows(g, mo, cap=max(fx["count"], 1))
    assert n_total == fx["count"] and r == fx["rows"]


# -------------------------------------------------- random tiny graphs vs oracle
@pytest.mark.parametrize("seed", range(8))
def test_tiny_random_vs_oracle(seed):
    rng = random.Random(seed)
    for k in range(25):
        L = rng.choice([1, 2, 3, 3, 4, 5])
        motif = rng.choice([c for c in CATALOG if len(c) == L] + [random_motif(rng, L)])
        src, dst, t, n = synth.tiny_graph(seed * 100 + k, n=rng.randint(2, 9), m=rng.randint(0, 90),
                                          tmax=rng.choice([5, 30, 200]))
        delta = rng.choice([0, 3, 10, 25, 100, INF])
        check_case(src, dst, t, n, motif, delta, random_fine(rng, L))


def test_tiny_vs_brute_directly():
    rng = random.Random(99)
    for k in range(20):
        motif = rng.choice(CATALOG)
        src, dst, t, n = synth.tiny_graph(7000 + k, n=6, m=50, tmax=30)
        delta = rng.choice([5, 15])
        g = T.Graph(src, dst, t, n)
        r, _ = gpu_rows(g, T.Motif(motif, delta))
        assert r == brute(src, dst, t, motif, delta)


def test_six_edge_and_seven_vertex_motifs():
    rng = random.Random(3)
    for k in range(10):
        motif = random_motif(rng, 6, max_v=7)
        src, dst, t, n = synth.tiny_graph(8000 + k, n=8, m=120, tmax=60)
        check_case(src, dst, t, n, motif, rng.choice([20, 60]), None)


def test_many_windows_spanning_tiles():
    """Windows longer than a 32-candidate batch, hub vertices, duplicate
    timestamps: C1-sized graph with a dense hub."""
    rng = np.random.default_rng(5)
    m, n = 6000, 40
    src = rng.integers(0, n, m).astype(np.uint32)
    dst = rng.integers(0, n, m).astype(np.uint32)
    hub = rng.random(m) < 0.3
    src[hub] = 0
    t = np.sort(rng.integers(0, 3000, m)).astype(np.int64)
    for motif in (M.TRI, M.STAR3, M.C4, [(0, 1), (1, 0), (0, 1)], M.TT):
        check_case(src, dst, t, n, motif, 40, None, rows=len(motif) <= 3)
        check_case(src, dst, t, n, motif, 40, [10] * (len(motif) - 1), rows=False)


# ----------------------------------------------------------------- edge cases
def test_edge_cases():
    e = np.zeros(0, np.uint32)
    g = T.Graph(e, e, np.zeros(0, np.int64), 4)
    assert T.tm_count(g, T.Motif(M.TRI, 10)) == 0
    rows, nt = T.tm_enumerate(g, T.Motif(M.TRI, 10), 4)
    assert nt == 0 and len(rows) == 0
    # all self-loops
    g = T.Graph(np.array([1, 1, 2]), np.array([1, 1, 2]), np.array([0, 1, 2]), 3)
    assert T.tm_count(g, T.Motif([(0, 1)], 10)) == 0
    # single edge motif = non-self-loop edges; root range restriction
    src, dst, t, n = synth.tiny_graph(1, n=5, m=300, tmax=100, p_self=0.2)
    g = T.Graph(src, dst, t, n)
    assert T.tm_count(g, T.Motif([(0, 1)], 0)) == int(np.sum(src != dst))
    S, D, _, _ = sorted_edges(src, dst, t)
    assert T.tm_count(g, T.Motif([(0, 1)], 0), root_range=(10, 50)) == sum(S[i] != D[i] for i in range(10, 50))
    assert T.tm_count(g, T.Motif(M.TRI, 30), root_range=(300, 400)) == 0
    # truncated enumeration: exact total, TM_TRUNCATED swallowed by the binding
    mo = T.Motif(M.TRI, 50)
    full = T.tm_count(g, mo)
    assert full > 4
    rows, nt = T.tm_enumerate(g, mo, 3)
    assert nt == full and len(rows) == 3
    Sx, Dx, Tx, _ = sorted_edges(src, dst, t)
    assert all(verify_match(Sx, Dx, Tx, M.TRI, 50, None, tuple(int(x) for x in r)) for r in rows)
    # δ = ∞ with fine bounds only
    check_case(src[:80], dst[:80], t[:80], n, M.C4, INF, [7, 7, 7], rows=False)


def test_sorted_view_and_input_order():
    src, dst, t, n = synth.tiny_graph(12, n=6, m=200, tmax=40)
    g = T.Graph(src, dst, t, n)
    S, D, Tt, order = sorted_edges(src, dst, t)
    s2, d2, t2 = g.sorted_edges()
    assert list(s2) == S and list(d2) == D and list(t2) == Tt
    assert list(g.sorted_to_input()) == order


def test_device_input_and_device_buffers():
    import torch
    src, dst, t, n = synth.config_graph("C1")
    dev = torch.device("cuda:0")
    g = T.Graph(torch.from_numpy(src.astype(np.int32)).to(dev), torch.from_numpy(dst.astype(np.int32)).to(dev),
                torch.from_numpy(t).to(dev), n)
    mo = T.Motif(M.TRI, 3600)
    exp = oracle.Graph(src, dst, t, n).mine(M.TRI, 3600, enumerate_=True)
    s = torch.cuda.Stream()
    assert T.tm_count(g, mo, stream=s) == exp["count"]
    buf = torch.zeros((exp["count"], 3), dtype=torch.int32, device=dev)
    rows, nt = T.tm_enumerate(g, mo, exp["count"], buf=buf, canonical=True)
    assert nt == exp["count"]
    assert np.array_equal(buf.cpu().numpy().astype(np.uint32), exp["rows"])
    roots = torch.arange(0, len(src), 7, dtype=torch.int64, device=dev)
    pr = T.tm_count_roots(g, mo, roots)
    opr = oracle.Graph(src, dst, t, n).mine(M.TRI, 3600, roots=np.arange(0, len(src), 7, dtype=np.uint64),
                                            per_root=True)["per_root"]
    assert np.array_equal(pr.cpu().numpy().astype(np.uint64), opr)


def test_shuffled_input_sorts_stably():
    src, dst, t, n = synth.config_graph("C1", shuffle=True)
    check_case(src, dst, t, n, M.TRI, 3600, None, roots=False)


# --------------------------------------------------------------- configs
def test_C1_count_and_enumerate():
    src, dst, t, n = synth.config_graph("C1")
    check_case(src, dst, t, n, M.TRI, 3600, None)


def test_C2_all_36_and_closed_forms():
    src, dst, t, n = synth.config_graph("C2")
    og = oracle.Graph(src, dst, t, n)
    g = T.Graph(src, dst, t, n)
    counts = []
    for name in M.CONFIG_MOTIFS["C2"]:
        mo = M.get(name)
        c = T.tm_count(g, T.Motif(mo, 3600))
        assert c == og.mine(mo, 3600)["count"], name
        counts.append(c)
    # invariants computed on the GPU alone, on a sub-graph the pure-Python
    # closed forms can evaluate
    s, d, tt = src[:4000], dst[:4000], t[:4000]
    gs = T.Graph(s, d, tt, n)
    assert sum(T.tm_count(gs, T.Motif(mm, 3600)) for mm in M.TWO_NODE) == two_node_closed_form(s, d, tt, 3600)
    s, d, tt = src[:1500], dst[:1500], t[:1500]
    gs = T.Graph(s, d, tt, n)
    assert sum(T.tm_count(gs, T.Motif(mm, 600)) for mm in M.P36) == census36_sum(s, d, tt, 600)


def test_C3_counts_vs_oracle():
    src, dst, t, n = synth.config_graph("C3")
    og = oracle.Graph(src, dst, t, n)
    g = T.Graph(src, dst, t, n)
    for name in M.CONFIG_MOTIFS["C3"]:
        mo = M.get(name)
        assert T.tm_count(g, T.Motif(mo, 86400)) == og.mine(mo, 86400)["count"], name


def test_C3_enumeration_full():
    src, dst, t, n = synth.config_graph("C3")
    og = oracle.Graph(src, dst, t, n)
    g = T.Graph(src, dst, t, n)
    mo = T.Motif(M.C4, 86400)
    exp = og.mine(M.C4, 86400, enumerate_=True)
    r, nt = gpu_rows(g, mo)
    assert nt == exp["n_total"]
    assert np.array_equal(np.array(r, np.uint32).reshape(-1, 4), exp["rows"])


def test_C4_full_size_sampled_roots_and_symmetry():
    """BASELINE config C4 at full size in the launch configuration bench.py
    times: per-root counts of 2^14 sampled roots vs the oracle, the full
    counts vs a time-reversed + direction-reversed copy of the graph."""
    src, dst, t, n = synth.config_graph("C4")
    g = T.Graph(src, dst, t, n)
    og = oracle.Graph(src, dst, t, n)
    rng = np.random.default_rng(0)
    roots = np.sort(rng.choice(len(src), 1 << 14, replace=False)).astype(np.uint64)
    full = {}
    for name in M.CONFIG_MOTIFS["C4"]:
        mot = M.get(name)
        fine = [21600] * (len(mot) - 1)
        mo = T.Motif(mot, 86400, fine)
        pr = T.tm_count_roots(g, mo, roots)
        assert np.array_equal(pr, og.mine(mot, 86400, fine, roots=roots, per_root=True)["per_root"]), name
        full[name] = T.tm_count(g, mo)
        # the sampled roots' counts agree with the count over the same roots in the timed kernel
    # time + direction reversal of the whole graph (sorted ids reversed)
    S, D, Tt = g.sorted_edges()
    C = int(Tt.max())
    gr = T.Graph(S[::-1].copy(), D[::-1].copy(), (C - Tt[::-1]).copy(), n)
    for name in M.CONFIG_MOTIFS["C4"]:
        mot = M.get(name)
        if not reverse_prefix_connected(mot):
            continue
        fine = [21600] * (len(mot) - 1)
        assert T.tm_count(gr, T.Motif(list(reversed(mot)), 86400, fine)) == full[name], name


def test_partition_slices_sum_to_full_count():
    """Multi-GPU plan exercised on one GPU: each rank's slice [lo, edge_hi)
    mined for its roots only sums to the unpartitioned count."""
    src, dst, t, n = synth.config_graph("C3")
    g = T.Graph(src, dst, t, n)
    S, D, Tt = g.sorted_edges()
    for mot, delta in ((M.TRI, 86400), (M.C4, 86400)):
        total = T.tm_count(g, T.Motif(mot, delta))
        for P in (2, 3, 8):
            lo, hi = T.tm_partition_plan(Tt, delta, P)
            s = 0
            for p in range(P):
                a, b, e = int(lo[p]), int(lo[p + 1]), int(hi[p])
                gp = T.Graph(S[a:e], D[a:e], Tt[a:e], n)
                s += T.tm_count(gp, T.Motif(mot, delta), root_range=(0, b - a))
            assert s == total


def test_generic_and_specialised_kernels_agree():
    src, dst, t, n = synth.config_graph("C1")
    g = T.Graph(src, dst, t, n)
    allr = np.arange(len(src), dtype=np.uint64)
    for mot in (M.TRI, M.TT, M.DIA, M.P36[7]):
        mo = T.Motif(mot, 3600)
        assert mo.specialised
        assert T.tm_count(g, mo) == int(T.tm_count_roots(g, mo, allr).sum())  # roots mode = generic kernel


def test_bursts_and_equal_timestamps():
    """Long runs of equal timestamps (horizon blocks whose answer range
    overflows the shared-memory stage) and sparse stretches."""
    rng = np.random.default_rng(21)
    m, n = 12000, 30
    src = rng.integers(0, n, m).astype(np.uint32)
    dst = rng.integers(0, n, m).astype(np.uint32)
    t = np.concatenate([np.full(5000, 100), np.sort(rng.integers(101, 100000, 2000)), np.full(5000, 200000)])
    t = t.astype(np.int64)
    for motif, delta, fine in ((M.TRI, 0, None), (M.PATH2, 50, None), (M.C4, 500, [0, 100, 100]),
                               (M.STAR3, 1000, None)):
        check_case(src, dst, t, n, motif, delta, fine, rows=False, roots=False)


# ------------------------------------------- heavy-subtree sharing (§8 a8)
@pytest.mark.parametrize("share", [0, 1, 2])
def test_heavy_subtree_sharing(share):
    """Skewed graph (two dense bursts own most of the search work):
    every sharing mode (0 on, 1 off, 2 eager) gives the oracle's counts,
    per-root counts, enumeration and search-tree counters, and the sharing
    modes really hand subtrees over."""
    src, dst, t, n = synth.burst_graph(231002806)
    og = oracle.Graph(src, dst, t, n)
    g = T.Graph(src, dst, t, n)
    allr = np.arange(len(src), dtype=np.uint64)
    shared = 0
    cases = [("TRI", None), ("C4", None), ("P3", [600, 600]), ("DIA", [None, 900, None, 1800]),
             ("TT", None)]
    for name, fine in cases:
        motif = M.get(name)
        exp = og.mine(motif, 3600, fine, enumerate_=True)
        mo = T.Motif(motif, 3600, fine)
        assert T.tm_count(g, mo, share=share) == exp["count"], name
        shared += T.tm_last_run_info()["shared_tasks"]
        rows, n_total = T.tm_enumerate(g, mo, exp["count"], canonical=True, share=share)
        shared += T.tm_last_run_info()["shared_tasks"]
        assert n_total == exp["n_total"]
        assert np.array_equal(rows, np.asarray(exp["rows"], np.uint32).reshape(-1, len(motif)))
        pr = og.mine(motif, 3600, fine, roots=allr, per_root=True)["per_root"]
        assert np.array_equal(T.tm_count_roots(g, mo, allr, share=share), pr), name
        st = T.tm_search_stats_run(g, mo, share=share)
        assert st["nodes"][:len(motif)] == exp["stats"]["nodes"][:len(motif)]
        assert st["window_sum"] == exp["stats"]["window_sum"]
    if share == 1:
        assert shared == 0
    elif share == 2:   # eager: hands over even short windows, so this small graph exercises it
        assert shared > 0


def test_sharing_rejects_bad_mode():
    g = T.Graph(np.array([0, 1], np.uint32), np.array([1, 2], np.uint32), np.array([0, 1], np.int64), 3)
    mo = T.Motif(M.get("P3")[:2], 10)
    with pytest.raises(T.TMotifError):
        T.tm_count(g, mo, share=3)


# ------------------------------------------------ fused 36-motif census (N1)
def test_census36_C2_vs_oracle():
    """tm_census36 on config C2 equals the oracle's 36 per-motif counts
    (bit-exact), whole graph and as a sum over root ranges."""
    src, dst, t, n = synth.config_graph("C2")
    og = oracle.Graph(src, dst, t, n)
    g = T.Graph(src, dst, t, n)
    exp = np.array([og.mine(M.P36[k], 3600)["count"] for k in range(36)], np.uint64)
    got = T.tm_census36(g, 3600)
    assert np.array_equal(got, exp)
    cuts = [0, 1000, 150_000, 150_001, len(src)]
    parts = sum(T.tm_census36(g, 3600, root_range=(cuts[i], cuts[i + 1])) for i in range(len(cuts) - 1))
    assert np.array_equal(parts, exp)
    # with per-gap bounds, against the oracle's fine-δ counts
    fine = [600, 1800]
    exp_f = np.array([og.mine(M.P36[k], 3600, fine)["count"] for k in range(36)], np.uint64)
    assert np.array_equal(T.tm_census36(g, 3600, fine), exp_f)


@pytest.mark.parametrize("seed", range(6))
def test_census36_tiny_random_vs_oracle(seed):
    rng = random.Random(1000 + seed)
    for k in range(12):
        src, dst, t, n = synth.tiny_graph(seed * 50 + k, n=rng.randint(2, 7), m=rng.randint(0, 120),
                                          tmax=rng.randint(5, 60))
        delta = rng.choice([0, 3, 10, 25, INF])
        fine = None if rng.random() < 0.4 else [rng.choice([0, 2, 7, INF]), rng.choice([0, 4, 12, INF])]
        og = oracle.Graph(src, dst, t, n)
        g = T.Graph(src, dst, t, n)
        exp = np.array([og.mine(M.P36[i], delta, fine)["count"] for i in range(36)], np.uint64)
        assert np.array_equal(T.tm_census36(g, delta, fine), exp), (seed, k, delta, fine)
        # and against the per-motif CUDA path
        if k % 4 == 0:
            got = [T.tm_count(g, T.Motif(M.P36[i], delta, fine)) for i in range(36)]
            assert np.array_equal(np.array(got, np.uint64), exp)


def test_census36_bursts_and_errors():
    src, dst, t, n = synth.burst_graph(231002807, n=300, m_bg=3000, core=24)
    og = oracle.Graph(src, dst, t, n)
    g = T.Graph(src, dst, t, n)
    exp = np.array([og.mine(M.P36[i], 3600)["count"] for i in range(36)], np.uint64)
    assert np.array_equal(T.tm_census36(g, 3600), exp)
    with pytest.raises(T.TMotifError):
        T.tm_census36(g, -1)
    empty = T.Graph(np.zeros(0, np.uint32), np.zeros(0, np.uint32), np.zeros(0, np.int64), 4)
    assert not T.tm_census36(empty, 10).any()


# ------------------------------------------- several motifs in one query
def test_count_multi_matches_single_queries_and_oracle():
    """tm_count_multi shares the horizons and window-end ranks across motifs
    with equal or different δ / δ_i; every count equals its own tm_count and
    the oracle's."""
    src, dst, t, n = synth.config_graph("C3", m=400_000)
    og = oracle.Graph(src, dst, t, n)
    g = T.Graph(src, dst, t, n)
    specs = [("P3", 86400, [21600, 21600]), ("TRI", 86400, [21600, 21600]), ("C4", 86400, [21600] * 3),
             ("DIA", 86400, [21600] * 4), ("TT", 3600, None), ("C4", 86400, [3600, None, 7200]),
             ("TT2", 43200, [43200, 600, 100000])]
    mos = [T.Motif(M.get(nm), d, f) for nm, d, f in specs]
    got = T.tm_count_multi(g, mos)
    info = T.tm_last_kernel_info()
    assert len(info) == len(specs) and all(x["mine_ms"] >= 0 for x in info)
    for (nm, d, f), mo, c in zip(specs, mos, got):
        assert c == T.tm_count(g, mo) == og.mine(M.get(nm), d, f)["count"], (nm, d, f)
    # root ranges and sharing modes pass through
    half = len(src) // 2
    assert T.tm_count_multi(g, mos, root_range=(half, len(src)), share=1) == \
        [og.mine(M.get(nm), d, f, root_range=(half, len(src)))["count"] for nm, d, f in specs]
    rng = random.Random(7)
    for k in range(30):
        s_, d_, t_, n_ = synth.tiny_graph(900 + k, n=rng.randint(2, 8), m=rng.randint(0, 80))
        ms = [M.get(rng.choice(["P3", "TRI", "C4", "TT", "DIA", "PATH2"])) for _ in range(rng.randint(1, 4))]
        dls = [rng.choice([0, 5, 20, INF]) for _ in ms]
        fs = [None if rng.random() < 0.5 else random_fine(rng, len(mm)) for mm in ms]
        gg = T.Graph(s_, d_, t_, n_)
        oo = oracle.Graph(s_, d_, t_, n_)
        res = T.tm_count_multi(gg, [T.Motif(mm, dd, ff) for mm, dd, ff in zip(ms, dls, fs)])
        assert res == [oo.mine(mm, dd, ff)["count"] for mm, dd, ff in zip(ms, dls, fs)]



# ------------------------------- generalized query: labels and anti-edges (N2)
def _cons_case(rng, motif, n_labels):
    verts = sorted({x for e in motif for x in e})
    vl = {v: rng.randrange(n_labels) for v in verts if rng.random() < 0.3} or None
    el = [rng.randrange(n_labels) if rng.random() < 0.25 else None for _ in motif]
    el = el if any(x is not None for x in el) else None
    anti = [tuple(rng.sample(verts, 2)) + (rng.randrange(len(motif)), rng.choice([0, 2, 5, 12, 40]))
            for _ in range(rng.choice([0, 1, 1, 2]))] or None
    return vl, el, anti


@pytest.mark.parametrize("seed", range(6))
def test_labels_and_anti_edges_tiny_vs_oracle(seed):
    """Counts, canonical enumeration, per-root counts and search-tree counters
    of generalized queries (labels + anti-edges) against the oracle."""
    rng = random.Random(5200 + seed)
    for k in range(25):
        n = rng.randint(2, 8)
        src, dst, t, _ = synth.tiny_graph(seed * 1000 + k, n=n, m=rng.randint(0, 90), tmax=rng.randint(4, 40))
        L = rng.choice([1, 2, 3, 3, 4, 5])
        motif = rng.choice([c for c in CATALOG if len(c) == L] + [random_motif(rng, L)])
        nl = rng.choice([1, 2, 3])
        vlab = [rng.randrange(nl) for _ in range(n)] if rng.random() < 0.7 else None
        elab = [rng.randrange(nl) for _ in range(len(src))] if rng.random() < 0.5 else None
        vl, el, anti = _cons_case(rng, motif, nl)
        delta = rng.choice([0, 3, 10, 25, INF])
        fine = random_fine(rng, L)
        og = oracle.Graph(src, dst, t, n)
        g = T.Graph(src, dst, t, n)
        if vlab is not None or elab is not None:
            og.set_labels(vlab, elab)
            g.set_labels(vlab, elab)
        exp = og.mine(motif, delta, fine, enumerate_=True, vlabels=vl, elabels=el, anti=anti)
        mo = T.Motif(motif, delta, fine, vlabels=vl, elabels=el, anti=anti)
        ctx = (seed, k, motif, delta, fine, vl, el, anti)
        assert T.tm_count(g, mo) == exp["count"], ctx
        rows, n_total = gpu_rows(g, mo)
        assert n_total == exp["n_total"], ctx
        assert rows == [tuple(int(x) for x in r) for r in exp["rows"]], ctx
        if len(src):
            allr = np.arange(len(src), dtype=np.uint64)
            pr = og.mine(motif, delta, fine, roots=allr, per_root=True, vlabels=vl, elabels=el, anti=anti)
            assert np.array_equal(T.tm_count_roots(g, mo, allr), pr["per_root"]), ctx
        st = T.tm_search_stats_run(g, mo)
        assert st["nodes"][:L] == exp["stats"]["nodes"][:L], ctx
        assert st["window_sum"] == exp["stats"]["window_sum"], ctx


def test_labels_and_anti_edges_at_scale():
    """A 400k-edge wiki-talk-shaped graph with 3 random vertex labels and 2
    edge labels: the Table 5 style V / V+T / V+T+A queries on the 4-cycle and
    the triangle against the oracle, through tm_count and tm_count_multi
    (which shares the anti-edge horizons with the motifs' own)."""
    src, dst, t, n = synth.config_graph("C3", m=400_000)
    rng = np.random.default_rng(5)
    vlab = rng.integers(0, 3, n).astype(np.int32)
    elab = rng.integers(0, 2, len(src)).astype(np.int32)
    og = oracle.Graph(src, dst, t, n)
    og.set_labels(vlab, elab)
    g = T.Graph(src, dst, t, n)
    g.set_labels(vlab, elab)
    day = 86400
    cases = [(M.C4, day, None, {0: 0, 2: 1}, None, None),                          # V
             (M.C4, day, [6 * 3600] * 3, {0: 0, 2: 1}, None, None),                # V+T
             (M.C4, day, [6 * 3600] * 3, {0: 0, 2: 1}, None, [(2, 0, 2, 3600)]),   # V+T+A (anti 2->0 on edge 2)
             (M.TRI, day, None, None, [1, None, 0], [(1, 0, 0, 7200), (0, 2, 2, 600)]),
             (M.P3, 3600, None, None, None, [(3, 0, 2, 1800)])]
    mos, exps = [], []
    for mot, d, f, vl, el, anti in cases:
        exp = og.mine(mot, d, f, vlabels=vl, elabels=el, anti=anti)["count"]
        mo = T.Motif(mot, d, f, vlabels=vl, elabels=el, anti=anti)
        assert T.tm_count(g, mo) == exp, (mot, d, f, vl, el, anti)
        mos.append(mo)
        exps.append(exp)
    assert T.tm_count_multi(g, mos) == exps
    # a device-side labelled copy (torch tensors) agrees
    import torch
    gd = T.Graph(torch.from_numpy(src.astype(np.int32)).cuda(), torch.from_numpy(dst.astype(np.int32)).cuda(),
                 torch.from_numpy(t).cuda(), n)
    gd.set_labels(torch.from_numpy(vlab).cuda(), torch.from_numpy(elab).cuda())
    assert T.tm_count(gd, mos[2]) == exps[2]


def test_generalized_query_errors():
    g = T.Graph(np.array([0, 1], np.uint32), np.array([1, 2], np.uint32), np.array([0, 1], np.int64), 3)
    with pytest.raises(T.TMotifError):
        T.Motif(M.P3, 10, anti=[(0, 0, 0, 5)])
    with pytest.raises(T.TMotifError):
        T.Motif(M.P3, 10, anti=[(0, 9, 0, 5)])
    with pytest.raises(T.TMotifError):
        T.Motif(M.P3, 10, anti=[(0, 1, 3, 5)])
    with pytest.raises(T.TMotifError):
        T.Motif(M.P3, 10, anti=[(0, 1, 0, -1)])
    with pytest.raises(T.TMotifError):
        T.Motif(M.P3, 10, vlabels={7: 1})
    with pytest.raises(T.TMotifError):
        T.Motif(M.P3, 10, elabels=[0, 0, 0, 0])
    with pytest.raises(ValueError):
        g.set_labels([0, 1])


# ------------------------------------- runtime-specialised kernels (N3, NVRTC)
def test_runtime_specialisation_parity():
    """tm_motif_specialise compiles the kernel template for motifs outside the
    build-time catalog (and GEN variants for labels / anti-edges); results stay
    bit-exact against the oracle and the generic kernel."""
    src, dst, t, n = synth.config_graph("C3", m=300_000)
    og = oracle.Graph(src, dst, t, n)
    g = T.Graph(src, dst, t, n)
    rng = np.random.default_rng(9)
    vlab = rng.integers(0, 2, n).astype(np.int32)
    og.set_labels(vlab, None)
    g.set_labels(vlab, None)
    day = 86400
    cases = [([(0, 1), (1, 2), (2, 3), (0, 3)], day, None, {}),               # not in the catalog
             ([(0, 1), (0, 2), (2, 1), (1, 3)], day, [7200, None, 3600], {}),
             ([(0, 1), (1, 0), (0, 2)], 3600, None, {}),                        # a P36 motif (catalog)
             (M.C4, day, [21600] * 3, {"vlabels": {0: 1}, "anti": [(2, 0, 2, 3600)]}),   # catalog + constraints
             (M.TRI, day, None, {"elabels": None, "anti": [(1, 0, 0, 600)]})]
    for mot, d, f, cons in cases:
        exp = og.mine(mot, d, f, enumerate_=True, **cons)
        generic = T.Motif(mot, d, f, **cons)
        c_generic = T.tm_count(g, generic)
        mo = T.Motif(mot, d, f, **cons).specialise()
        assert mo.specialised
        assert T.tm_count(g, mo) == c_generic == exp["count"], (mot, cons)
        rows, n_total = gpu_rows(g, mo)
        assert n_total == exp["n_total"]
        assert rows == [tuple(int(x) for x in r) for r in exp["rows"]]
    # changing a constraint drops the specialisation (the kernel would not check it)
    mo = T.Motif([(0, 1), (1, 2), (2, 3), (0, 3)], day).specialise()
    assert mo.specialised
    T.lib().tm_motif_add_anti_edge(mo.handle, 3, 1, 0, 100)
    assert not mo.specialised


def test_prefix_fusion():
    """tm_count_multi counts a motif that is a prefix of another (same δ and
    gap bounds, no constraints) as that motif's level-l search-tree nodes:
    P3 inside C4, TRI inside DIA and TT, PATH2 inside everything — counts equal
    the unfused query and the oracle; a different δ_i or δ blocks the fusion."""
    src, dst, t, n = synth.config_graph("C3", m=300_000)
    og = oracle.Graph(src, dst, t, n)
    g = T.Graph(src, dst, t, n)
    d, f = 86400, 21600
    specs = [("P3", d, [f] * 2), ("C4", d, [f] * 3), ("TRI", d, [f] * 2), ("DIA", d, [f] * 4),
             ("TT", d, [f] * 3), ("PATH2", d, [f]), ("P3", d, [f, 3600]), ("TRI", 3600, [f] * 2),
             ("TRI", d, None), ("TT", d, None)]
    mos = [T.Motif(M.get(nm), dd, ff) for nm, dd, ff in specs]
    fused = T.tm_count_multi(g, mos)
    kin = T.tm_last_kernel_info()
    plain = T.tm_count_multi(g, mos, fuse=1)
    exp = [og.mine(M.get(nm), dd, ff)["count"] for nm, dd, ff in specs]
    assert fused == plain == exp
    carried = {i: x["carried_by"] for i, x in enumerate(kin) if x["carried_by"] >= 0}
    # P3/d/f in C4, TRI/d/f in C4 (sibling rows) or DIA (prefix), PATH2 in a longer motif,
    # TRI/d/None in TT/d/None
    assert set(carried) == {0, 2, 5, 8}, carried
    assert carried[0] == 1 and carried[2] in (1, 3) and carried[8] == 9
    assert all(kin[i]["grid_ctas"] == 0 for i in carried)


def test_prefix_fusion_generic_and_specialised_carriers():
    """Prefix fusion on the generic kernel (a carrier outside the catalog runs
    PlanR in the prefix-counting mode), several prefixes of one carrier
    (PATH2 and P3 inside one 4-edge motif), root ranges, sharing modes, and an
    NVRTC-specialised carrier (fusion declined, counts unchanged)."""
    src, dst, t, n = synth.config_graph("C3", m=200_000)
    og = oracle.Graph(src, dst, t, n)
    g = T.Graph(src, dst, t, n)
    d = 86400
    chord = [(0, 1), (1, 2), (2, 3), (0, 3)]          # not in the catalog
    specs = [(M.PATH2, d, None), (M.P3, d, None), (chord, d, None)]
    mos = [T.Motif(mm, dd, ff) for mm, dd, ff in specs]
    for rr in (None, (50_000, 150_000)):
        for share in (0, 1, 2):
            kw = {} if rr is None else {"root_range": rr}
            got = T.tm_count_multi(g, mos, share=share, **kw)
            exp = [og.mine(mm, dd, ff, **kw)["count"] for mm, dd, ff in specs]
            assert got == exp, (rr, share)
            kin = T.tm_last_kernel_info()
            assert kin[0]["carried_by"] == 2 and kin[1]["carried_by"] == 2 and kin[2]["carried_by"] == -1
    spec = T.Motif(chord, d).specialise()
    got = T.tm_count_multi(g, [T.Motif(M.P3, d), spec])
    assert got == [og.mine(M.P3, d)["count"], og.mine(chord, d)["count"]]
    assert [x["carried_by"] for x in T.tm_last_kernel_info()] == [-1, -1]


def test_sibling_rows_and_resume():
    """The 4-cycle kernel also writes the triangles it sees at level 2 (TRI is
    its sibling: same first two edges, its closing edge read from the same
    window); TRI's count is their number and the diamond resumes from them at
    level 3 — counts equal the oracle and the unfused query, also when the
    triangles overflow the row buffer (the diamond is then searched again)."""
    d, f = 86400, 21600
    src, dst, t, n = synth.config_graph("C3", m=300_000)
    og = oracle.Graph(src, dst, t, n)
    g = T.Graph(src, dst, t, n)
    sets = [[("C4", [f] * 3), ("TRI", [f] * 2), ("DIA", [f] * 4)],
            [("P3", [f] * 2), ("TRI", [f] * 2), ("C4", [f] * 3), ("DIA", [f] * 4)],
            [("TRI", None), ("C4", None)],
            [("DIA", [f] * 4), ("C4", [f] * 3), ("TT", [f] * 3), ("TRI", [f] * 2)]]
    for specs in sets:
        mos = [T.Motif(M.get(nm), d, ff) for nm, ff in specs]
        exp = [og.mine(M.get(nm), d, ff)["count"] for nm, ff in specs]
        assert T.tm_count_multi(g, mos) == exp, specs
        assert T.tm_count_multi(g, mos, fuse=1) == exp
    mos = [T.Motif(M.get(nm), d, ff) for nm, ff in sets[0]]
    T.tm_count_multi(g, mos)
    kin = T.tm_last_kernel_info()
    assert kin[1]["carried_by"] == 0 and kin[1]["grid_ctas"] == 0   # TRI: rows of the 4-cycle kernel
    assert kin[2]["grid_ctas"] > 0                                   # the diamond's resume kernel ran
    assert [x["kernel_mode"] for x in kin] == [T.KMODE_COUNT_SIB, T.KMODE_NONE, T.KMODE_RESUME]
    T.tm_count_multi(g, mos, fuse=1)
    assert [x["kernel_mode"] for x in T.tm_last_kernel_info()] == [T.KMODE_COUNT] * 3
    # dense bursts: thousands of triangles and diamonds (the row buffer holds them all)
    for core in (30, 40):
        s1, d1, t1, n1 = synth.burst_graph(11, n=2000, m_bg=20000, bursts=2, core=core, burst_len=1800)
        og1 = oracle.Graph(s1, d1, t1, n1)
        g1 = T.Graph(s1, d1, t1, n1)
        f1 = [1200] * 4
        specs = [("P3", f1[:2]), ("C4", f1[:3]), ("TRI", f1[:2]), ("DIA", f1), ("TT", f1[:3])]
        exp = [og1.mine(M.get(nm), 3600, ff)["count"] for nm, ff in specs]
        assert exp[2] > 5000 and exp[3] > 10000 and exp[2] < 65536
        mos1 = [T.Motif(M.get(nm), 3600, ff) for nm, ff in specs]
        assert T.tm_count_multi(g1, mos1) == exp
        kin = T.tm_last_kernel_info()
        assert kin[2]["carried_by"] == 1 and kin[3]["grid_ctas"] > 0 and kin[3]["carried_by"] == -1
    # overflow of the row buffer (65536 rows for a small graph): dense bursts
    s2, d2, t2, n2 = synth.burst_graph(7, n=2000, m_bg=5000, bursts=3, core=80, burst_len=900)
    og2 = oracle.Graph(s2, d2, t2, n2)
    g2 = T.Graph(s2, d2, t2, n2)
    specs = [("C4", None), ("TRI", None), ("DIA", None)]
    exp = [og2.mine(M.get(nm), 3600, ff)["count"] for nm, ff in specs]
    assert exp[1] > 65536
    assert T.tm_count_multi(g2, [T.Motif(M.get(nm), 3600, ff) for nm, ff in specs]) == exp


# ------------------------------------------- prefix-disconnected motifs (Q9)
DISCONNECTED = [[(0, 1), (2, 3)], [(0, 1), (2, 3), (1, 2)], [(0, 1), (2, 3), (3, 0)],
                [(0, 1), (2, 3), (4, 5)], [(0, 1), (1, 2), (3, 4), (4, 0)], [(0, 1), (2, 1), (3, 4)]]


@pytest.mark.parametrize("seed", range(3))
def test_disconnected_motifs_vs_oracle(seed):
    """AllEdges levels on the thread-per-root kernel: counts,
    enumerations and per-root counts equal the oracle's."""
    rng = random.Random(700 + seed)
    for k in range(18):
        motif = DISCONNECTED[k % len(DISCONNECTED)]
        src, dst, t, n = synth.tiny_graph(seed * 100 + k, n=rng.randint(4, 12), m=rng.randint(0, 80), tmax=40)
        delta = rng.choice([0, 3, 10, INF])
        check_case(src, dst, t, n, motif, delta, random_fine(rng, len(motif)), stats=False)
    # a bigger graph: several thousand roots, long all-edge windows
    src, dst, t, n = synth.config_graph("C1", m=3000)
    for motif, delta in (([(0, 1), (2, 3)], 600), ([(0, 1), (2, 3), (1, 2)], 7200), ([(0, 1), (1, 2), (3, 4), (4, 0)], 20000)):
        c = check_case(src, dst, t, n, motif, delta, None, rows=seed == 0, stats=False)
        assert c > 0


def test_disconnected_in_multi_and_errors():
    src, dst, t, n = synth.config_graph("C1", m=2000)
    og = oracle.Graph(src, dst, t, n)
    g = T.Graph(src, dst, t, n)
    specs = [([(0, 1), (2, 3)], 7200), (M.P3, 7200), ([(0, 1), (2, 3), (1, 2)], 7200), (M.TRI, 7200)]
    exp = [og.mine(mm, d)["count"] for mm, d in specs]
    assert T.tm_count_multi(g, [T.Motif(mm, d) for mm, d in specs]) == exp
    kin = T.tm_last_kernel_info()
    assert kin[0]["kernel_mode"] == T.KMODE_DFS and kin[2]["kernel_mode"] == T.KMODE_DFS
    mo = T.Motif([(0, 1), (2, 3)], 600)
    with pytest.raises(T.TMotifError) as e:
        T.tm_search_stats_run(g, mo)
    assert e.value.status == T.TM_EUNSUPPORTED
    with pytest.raises(T.TMotifError) as e:
        T.tm_count(g, T.Motif([(0, 1), (2, 3)], 600, vlabels={0: 1}))
    assert e.value.status == T.TM_EUNSUPPORTED


# ------------------------------------- the timed configuration
C4_BENCH = [("P3", [21600] * 2), ("TRI", [21600] * 2), ("C4", [21600] * 3), ("DIA", [21600] * 4)]


def _bench_query(delta=86400):
    return [T.Motif(M.get(nm), delta, f) for nm, f in C4_BENCH]


def test_C4_bench_query_full_oracle():
    """bench.py's exact timed query — tm_count_multi over P3/TRI/C4/DIA at
    δ = 1 d, δ_i = 6 h on the full 63.5M-edge C4 graph, fused (the 4-cycle
    kernel in kCountSib mode counting P3 as its level-3 nodes and writing TRI's
    rows, the diamond resumed from those rows) — equals the full oracle count
    of every motif (exact), and equals the unfused query."""
    src, dst, t, n = synth.config_graph("C4")
    g = T.Graph(src, dst, t, n)
    got = T.tm_count_multi(g, _bench_query())
    modes = [x["kernel_mode"] for x in T.tm_last_kernel_info()]
    assert modes == [T.KMODE_NONE, T.KMODE_NONE, T.KMODE_COUNT_SIB, T.KMODE_RESUME], modes
    og = oracle.Graph(src, dst, t, n)
    exp = [og.mine(M.get(nm), 86400, f)["count"] for nm, f in C4_BENCH]
    assert got == exp, (got, exp)
    assert T.tm_count_multi(g, _bench_query(), fuse=1) == exp


@pytest.mark.parametrize("cfg", ["C3", "C4"])
def test_specialised_kernels_root_subranges(cfg):
    """Per-root parity of the kernels bench.py times (the catalog's
    specialised PlanC kernels in the kCount / kCountSib / kCountPfx / kResume
    modes, not the generic per-root PlanR kernel): 64 random root sub-ranges,
    each a separate tm_count_multi / tm_count, against the oracle's count over
    the same roots."""
    src, dst, t, n = synth.config_graph(cfg)
    m = len(src)
    g = T.Graph(src, dst, t, n)
    og = oracle.Graph(src, dst, t, n)
    rng = np.random.default_rng(64)
    mos = _bench_query()
    for k in range(64):
        w = int(rng.choice([1, 37, 1000, 20000]))
        lo = int(rng.integers(0, m - w))
        rr = (lo, lo + w)
        got = T.tm_count_multi(g, mos, root_range=rr)
        exp = [og.mine(M.get(nm), 86400, f, root_range=rr)["count"] for nm, f in C4_BENCH]
        assert got == exp, (cfg, rr, got, exp)
        if k % 8 == 0:   # the plain specialised counting kernel, one motif per query
            for (nm, f), mo, e in zip(C4_BENCH, mos, exp):
                assert mo.specialised
                assert T.tm_count(g, mo, root_range=rr) == e, (cfg, rr, nm)


def test_fusion_keeps_sibling_carrier():
    """a motif that writes a sibling's rows (the 4-cycle
    for TRI) must keep its own kernel even when a longer motif (a 5-edge
    extension of the 4-cycle) could count it as a prefix — otherwise TRI
    (and the motifs resuming from its rows) read 0."""
    d, f = 3600, 1200
    src, dst, t, n = synth.burst_graph(11, n=2000, m_bg=20000, bursts=2, core=30, burst_len=1800)
    og = oracle.Graph(src, dst, t, n)
    g = T.Graph(src, dst, t, n)
    c4x = M.C4 + [(0, 2)]
    sets = [[(M.C4, [f] * 3), (M.TRI, [f] * 2), (c4x, [f] * 4)],
            [(M.C4, None), (M.TRI, None), (c4x, None), (M.DIA, None)],
            [(c4x, [f] * 4), (M.DIA, [f] * 4), (M.TRI, [f] * 2), (M.C4, [f] * 3), (M.P3, [f] * 2)]]
    for specs in sets:
        mos = [T.Motif(mm, d, ff) for mm, ff in specs]
        exp = [og.mine(mm, d, ff)["count"] for mm, ff in specs]
        assert all(e > 0 for e in exp)
        assert T.tm_count_multi(g, mos) == exp, specs
        assert T.tm_count_multi(g, mos, fuse=1) == exp, specs


# --------------------------------------- hardening and invariants
@pytest.mark.timeout(300)
def test_concurrent_sharing_kernels_on_two_streams():
    """tmotif.h allows concurrent tm_count calls on different streams.  The
    heavy-subtree sharing kernels need every CTA resident (idle warps wait for
    hand-overs), so they launch cooperatively: two of them started from two
    host threads on two streams, each filling the GPU, must both finish with
    the oracle's counts (no partial residency deadlock)."""
    import threading
    import torch
    src, dst, t, n = synth.burst_graph(231002806)
    og = oracle.Graph(src, dst, t, n)
    g = T.Graph(src, dst, t, n)
    cases = [(M.C4, None), (M.TT, None), (M.TRI, None), (M.P3, [600, 600])]
    exp = [og.mine(mm, 3600, f)["count"] for mm, f in cases]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    out = [[None] * len(cases) for _ in range(2)]
    errs = []

    def worker(k):
        try:
            for rep in range(3):
                for i, (mm, f) in enumerate(cases):
                    out[k][i] = T.tm_count(g, T.Motif(mm, 3600, f), stream=streams[k], share=2 if k else 0)
        except Exception as ex:   # surfaced below
            errs.append(ex)

    th = [threading.Thread(target=worker, args=(k,)) for k in range(2)]
    for x in th:
        x.start()
    for x in th:
        x.join(timeout=240)
    assert not any(x.is_alive() for x in th), "concurrent sharing kernels did not finish"
    assert not errs, errs
    assert out[0] == exp and out[1] == exp


def test_C4_delta_sweeps_monotone():
    """SURVEY §8(c) pin 2 at config scale, on the GPU alone: the bench query's
    counts never decrease as δ grows (δ_i fixed) or as every δ_i grows
    (δ fixed), and δ_i >= δ equals the coarse-only query."""
    src, dst, t, n = synth.config_graph("C4")
    g = T.Graph(src, dst, t, n)
    prev = None
    for d in (0, 3600, 21600, 43200, 86400, 2 * 86400):
        c = T.tm_count_multi(g, [T.Motif(M.get(nm), d, f) for nm, f in C4_BENCH])
        if prev is not None:
            assert all(a <= b for a, b in zip(prev, c)), (d, prev, c)
        prev = c
    prev = None
    for fi in (0, 600, 3600, 21600, 86400):
        c = T.tm_count_multi(g, [T.Motif(M.get(nm), 86400, [fi] * (len(M.get(nm)) - 1)) for nm, _ in C4_BENCH])
        if prev is not None:
            assert all(a <= b for a, b in zip(prev, c)), (fi, prev, c)
        prev = c
    coarse = T.tm_count_multi(g, [T.Motif(M.get(nm), 86400) for nm, _ in C4_BENCH])
    assert prev == coarse   # δ_i = δ: the gap bounds are implied by the window


def test_C4_bench_query_partitions_agree():
    """SURVEY §8(c) pin 2 / §8(e): the bench query split for 1, 2, 4 and 8
    ranks — contiguous root ranges from tm_partition_plan, each rank's slice
    (roots + forward δ-halo) built as its own graph and mined
    fused — sums to the same counts (a match belongs to the rank holding e_1)."""
    src, dst, t, n = synth.config_graph("C4")
    g = T.Graph(src, dst, t, n)
    S, D, Tt = g.sorted_edges()
    g.close()
    from paper_2310_02800_b200 import multi
    reach = max(multi.reach(86400, f) for _, f in C4_BENCH)
    totals = []
    for P in (1, 2, 4, 8):
        acc = np.zeros(len(C4_BENCH), np.int64)
        for r in range(P):
            a, b, e = multi.rank_slice(Tt, reach, P, r)
            gp = T.Graph(S[a:e], D[a:e], Tt[a:e], n)
            acc += np.array(T.tm_count_multi(gp, _bench_query(), root_range=(0, b - a)), np.int64)
            gp.close()
        totals.append(acc.tolist())
    assert all(x == totals[0] for x in totals), totals


def test_C5_slice_sampled_roots_specialised():
    """BASELINE configs[4] (C5, 2e9 edges) is mined as time slices with δ-halos:
    on one slice, 16 random root ranges of 4096 roots (2^16 roots) through the
    specialised fused kernels the C5 bench times (TRI as the 4-cycle's sibling
    rows) against the oracle over the same roots, and the slice's full count
    against the generic kernel's per-root counts."""
    s, d, t, n, nr = synth.c5_rank_slice(3, 64, 3600)
    g = T.Graph(s, d, t, n)
    og = oracle.Graph(s, d, t, n)
    mos = [T.Motif(M.TRI, 3600), T.Motif(M.C4, 3600)]
    rng = np.random.default_rng(5)
    for _ in range(16):
        lo = int(rng.integers(0, nr - 4096))
        rr = (lo, lo + 4096)
        got = T.tm_count_multi(g, mos, root_range=rr)
        assert [x["kernel_mode"] for x in T.tm_last_kernel_info()] == [T.KMODE_NONE, T.KMODE_COUNT_SIB]
        exp = [og.mine(mm, 3600, root_range=rr)["count"] for mm in (M.TRI, M.C4)]
        assert got == exp, (rr, got, exp)
    full = T.tm_count_multi(g, mos, root_range=(0, nr))
    allr = np.arange(nr, dtype=np.uint64)
    assert full == [int(T.tm_count_roots(g, mo, allr).sum()) for mo in mos]


def test_wide_timestamp_ranges():
    """Horizons in nanosecond-like units: a block's staged timestamp range can
    span more than 2^32 units (u32 offsets cannot hold it; the horizon kernel
    then searches global memory) next to blocks that fit — counts, per-root
    counts and enumeration still equal the oracle's."""
    rng = np.random.default_rng(2024)
    m, n = 30000, 60
    src = rng.integers(0, n, m).astype(np.uint32)
    dst = rng.integers(0, n, m).astype(np.uint32)
    t = np.sort(rng.integers(0, 7 * 86400, m)).astype(np.int64) * 1_000_000_000   # seconds -> ns
    t[m // 2:] += 10 ** 15                                                           # a gap of ~11.6 days
    t[1000:1300] = t[1000]                                                            # a burst of equal times
    for motif, delta, fine, rows in ((M.TRI, 3600 * 10 ** 9, None, True),
                                     (M.C4, 7200 * 10 ** 9, [1800 * 10 ** 9] * 3, True),
                                     (M.P3, 20000 * 10 ** 9, None, False)):
        check_case(src, dst, t, n, motif, delta, fine, rows=rows, stats=False, roots=True)


def test_timed_kernel_node_counts_equal_algorithm1():
    """The candidate-caching invariant (every window is searched
    once, when its node is created) on the kernels the bench times, not only
    on the instrumentation replay: with PATH2 and P3 fused into the 4-cycle's
    kernel (kCountPfx counts the nodes it creates at levels 2 and 3), those
    counts equal the oracle's Algorithm 1 search-tree node counts of the
    4-cycle search, level by level (C3 and C4, with and without gap bounds)."""
    for cfg, delta, f in (("C3", 86400, None), ("C4", 86400, 21600)):
        src, dst, t, n = synth.config_graph(cfg)
        g = T.Graph(src, dst, t, n)
        og = oracle.Graph(src, dst, t, n)
        fine = lambda L: None if f is None else [f] * (L - 1)   # noqa: E731
        got = T.tm_count_multi(g, [T.Motif(M.PATH2, delta, fine(2)), T.Motif(M.P3, delta, fine(3)),
                                   T.Motif(M.C4, delta, fine(4))])
        info = T.tm_last_kernel_info()
        assert info[0]["carried_by"] == 2 and info[1]["carried_by"] == 2, info
        st = og.mine(M.C4, delta, fine(4))["stats"]
        assert got[0] == st["nodes"][2] and got[1] == st["nodes"][3], (cfg, got, st["nodes"])
        assert got[2] == st["matches"]


def test_pair_index_long_closing_windows():
    """tm_graph_opts.pair_index: closing edges whose window in a hub's list runs
    past the in-lane scan are counted from the pair index (two binary searches
    over the pair's edges).  On a skewed graph (dense bursts: long hub windows)
    counts and per-root counts equal the oracle's with and without gap bounds
    (known and unknown window ends), through the specialised and the generic
    kernels, and the fused C5 query on a C5 slice equals the query without the
    index."""
    src, dst, t, n = synth.burst_graph(231002806)
    og = oracle.Graph(src, dst, t, n)
    g = T.Graph(src, dst, t, n, pair_index=True)
    allr = np.arange(len(src), dtype=np.uint64)
    for name, fine in (("C4", None), ("C4", [900, 900, 900]), ("TRI", None), ("TT2", None),
                       ("DIA", [None, 900, None, 1800]), ("P3", None)):
        motif = M.get(name)
        mo = T.Motif(motif, 3600, fine)
        exp = og.mine(motif, 3600, fine)["count"]
        assert T.tm_count(g, mo) == exp, name
        pr = og.mine(motif, 3600, fine, roots=allr, per_root=True)["per_root"]
        assert np.array_equal(T.tm_count_roots(g, mo, allr), pr), name
    s, d, tt, nn, nr = synth.c5_rank_slice(5, 64, 3600)
    mos = [T.Motif(M.TRI, 3600), T.Motif(M.C4, 3600)]
    with_idx = T.tm_count_multi(T.Graph(s, d, tt, nn, pair_index=True), mos, root_range=(0, nr))
    without = T.tm_count_multi(T.Graph(s, d, tt, nn), mos, root_range=(0, nr))
    assert with_idx == without and with_idx[1] > 0


def test_next_id_cache_repeated_and_concurrent_queries():
    """The first query that builds window descriptors for a list variant
    records each edge's first-record id in that list (a δ-independent graph
    index, NextIdCache); later queries on the graph skip the record read of
    windows ending before it.  Queries before and after it is recorded, with
    other gap bounds, and first queries racing on two streams of fresh graphs
    all equal the oracle."""
    import threading
    import torch
    src, dst, t, n = synth.config_graph("C3", m=400_000)
    og = oracle.Graph(src, dst, t, n)
    cases = [(M.P3, [1800, 1800]), (M.C4, [3600] * 3), (M.TRI, [600, 600]), (M.DIA, [7200] * 4),
             (M.C4, [1800] * 3)]
    exp = [og.mine(mm, 86400, f)["count"] for mm, f in cases]
    g = T.Graph(src, dst, t, n)
    for rep in range(2):   # rep 0: the first C4-shaped query records the ids; rep 1: all use them
        assert [T.tm_count(g, T.Motif(mm, 86400, f)) for mm, f in cases] == exp, rep
    assert T.tm_count_multi(g, [T.Motif(mm, 86400, f) for mm, f in cases]) == exp
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for trial in range(3):
        g2 = T.Graph(src, dst, t, n)   # nothing recorded yet: both streams race to be first
        out = [None, None]
        errs = []

        def worker(k):
            try:
                out[k] = [T.tm_count(g2, T.Motif(mm, 86400, f), stream=streams[k]) for mm, f in cases[k::2]]
            except Exception as ex:   # surfaced below
                errs.append(ex)

        th = [threading.Thread(target=worker, args=(k,)) for k in range(2)]
        for x in th:
            x.start()
        for x in th:
            x.join(timeout=120)
        assert not errs, errs
        assert out[0] == exp[0::2] and out[1] == exp[1::2], trial


@pytest.mark.parametrize("k", [4, 6, 9])
def test_pair_bucket_filter_vs_oracle(k):
    """tm_graph_opts.pair_id_bucket_log2: closing leaves skip every pair with no
    edge in the (at most two) 2^k-id buckets their window covers, and fall back
    to the plain pair filter when the window covers more.  Small buckets force
    both paths on a skewed graph: counts and per-root counts equal the
    oracle's, with and without gap bounds, and the fused C5-slice query equals
    the query without any index."""
    src, dst, t, n = synth.burst_graph(231002806)
    og = oracle.Graph(src, dst, t, n)
    g = T.Graph(src, dst, t, n, pair_index=True, pair_id_bucket_log2=k)
    allr = np.arange(len(src), dtype=np.uint64)
    for name, fine in (("C4", None), ("C4", [900, 900, 900]), ("TRI", None), ("TT2", None), ("P3", None)):
        motif = M.get(name)
        mo = T.Motif(motif, 3600, fine)
        assert T.tm_count(g, mo) == og.mine(motif, 3600, fine)["count"], (k, name)
        pr = og.mine(motif, 3600, fine, roots=allr, per_root=True)["per_root"]
        assert np.array_equal(T.tm_count_roots(g, mo, allr), pr), (k, name)
    s, d, tt, nn, nr = synth.c5_rank_slice(5, 64, 3600)
    mos = [T.Motif(M.TRI, 3600), T.Motif(M.C4, 3600)]
    with_idx = T.tm_count_multi(T.Graph(s, d, tt, nn, pair_index=True, pair_id_bucket_log2=k + 10), mos,
                                root_range=(0, nr))
    without = T.tm_count_multi(T.Graph(s, d, tt, nn), mos, root_range=(0, nr))
    assert with_idx == without and with_idx[1] > 0


def test_C5_bench_slice_with_pair_filters_vs_oracle():
    """The exact C5 bench configuration: a 1/128 time slice built with the pair
    index and the id-bucketed pair filter (2^k >= 2 m δ / span, bench.py),
    mined by the fused TRI + 4-cycle query: 16 random ranges of 4096 roots
    equal the oracle over the same roots, and the whole slice equals the
    query on the same slice without any index."""
    import math
    s, d, t, n, nr = synth.c5_rank_slice(48, 128, 3600)
    span = max(1, int(t[-1]) - int(t[0]))
    k = max(1, int(math.ceil(math.log2(max(2.0 * len(t) * 3600 / span, 2.0)))))
    g = T.Graph(s, d, t, n, pair_index=True, pair_id_bucket_log2=k)
    og = oracle.Graph(s, d, t, n)
    mos = [T.Motif(M.TRI, 3600), T.Motif(M.C4, 3600)]
    rng = np.random.default_rng(128)
    for _ in range(16):
        lo = int(rng.integers(0, nr - 4096))
        rr = (lo, lo + 4096)
        got = T.tm_count_multi(g, mos, root_range=rr)
        exp = [og.mine(mm, 3600, root_range=rr)["count"] for mm in (M.TRI, M.C4)]
        assert got == exp, (k, rr, got, exp)
    full = T.tm_count_multi(g, mos, root_range=(0, nr))
    assert full == T.tm_count_multi(T.Graph(s, d, t, n), mos, root_range=(0, nr)) and full[1] > 0
