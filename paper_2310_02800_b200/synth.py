"""Seeded synthetic temporal graphs — the ONLY module shared by the oracle
side (tests/, bench.py's cpu_baseline) and the CUDA side.  It holds none of
the method's arithmetic: it only draws edges.

Shapes follow the paper's datasets (Table 3) as planned
in SURVEY.md §8(d) "Synthetic generator":

1. vertex activity ``w_i = (π(i)+1)^-α`` with π a seeded permutation, shares
   capped at ``cap`` (hubs both send and receive);
2. ``S ≈ m/μ`` *sessions* (μ = temporal/static edge ratio of the dataset):
   a pair (u~w, v~w, u≠v except a 0.1 % self-loop rate), a start
   ``s ~ U[0, span)``, ``Geom(1/μ)`` events (mean μ) at ``s + Σ Exp(β)``
   (integer seconds), each event reversed (v→u) with probability ``p_reply``;
3. email shape only: with probability ``fanout`` an event is copied to 1-4
   extra recipients at the **same timestamp** (exercises the tie rule Q1);
4. clip to the span, keep exactly ``m`` events in session order, order by
   ``(t, session, event)``.

All randomness comes from ``numpy.random.default_rng(seed)`` (PCG64), so a
config + seed fixes the graph bit for bit.  Seeds: ``231002800 + config``.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

DAY = 86400
YEAR = 365 * DAY
SEED_BASE = 231002800


@dataclasses.dataclass(frozen=True)
class GraphSpec:
    name: str
    n: int
    m: int
    span: int          # seconds
    mu: float          # mean events per session (temporal/static edge ratio)
    alpha: float       # power-law exponent of vertex activity
    cap: float         # max activity share of one vertex
    beta: float        # mean inter-event gap inside a session (s)
    fanout: float = 0.0
    p_reply: float = 0.3
    p_self: float = 0.001
    t0: int = 1_200_000_000   # epoch-like base time


# SURVEY.md §8(d) table (α, cap, β, p_reply are proposals, not paper values)
SPECS = {
    "C1": GraphSpec("C1 tiny", 1000, 20_000, 7 * DAY, 2.0, 1.0, 0.03, 3600.0),
    "C2": GraphSpec("C2 email-Eu-core-shaped", 986, 332_334, 803 * DAY, 13.3, 1.0, 0.03, 600.0, fanout=0.1),
    "C3": GraphSpec("C3 wiki-talk-shaped", 1_140_149, 7_833_140, int(6.24 * YEAR), 2.81, 1.0, 0.01, 3600.0),
    "C4": GraphSpec("C4 stackoverflow-shaped", 2_601_977, 63_497_050, int(7.6 * YEAR), 1.82, 1.0, 0.003, 3600.0),
}


def activity(n: int, alpha: float, cap: float, rng: np.random.Generator) -> np.ndarray:
    """Vertex sampling probabilities: (π(i)+1)^-α, shares clipped at ``cap``."""
    rank = rng.permutation(n).astype(np.float64)
    p = (rank + 1.0) ** (-alpha)
    p /= p.sum()
    if cap * n < 1.0:
        cap = 1.0 / n
    for _ in range(100):
        over = p > cap
        if not over.any():
            break
        excess = float((p[over] - cap).sum())
        p[over] = cap
        free = p < cap
        p[free] += excess * p[free] / p[free].sum()
    return p / p.sum()


def generate(spec: GraphSpec, seed: int, *, m: int | None = None, shuffle: bool = False):
    """Returns (src u32[m], dst u32[m], t i64[m], n).  Sorted by time unless
    ``shuffle`` (a seeded permutation of the input order)."""
    rng = np.random.default_rng(seed)
    n = spec.n
    m = spec.m if m is None else m
    p = activity(n, spec.alpha, spec.cap, rng)

    def draw(k):
        # k i.i.d. draws from p: multinomial counts, then a seeded shuffle
        return rng.permutation(np.repeat(np.arange(n, dtype=np.int64), rng.multinomial(k, p)))

    per_session = spec.mu * (1.0 + spec.fanout * 2.5)
    S = int(math.ceil(m / per_session * 1.15)) + 64
    u = draw(S)
    v = draw(S)
    for _ in range(16):
        bad = np.nonzero(u == v)[0]
        if bad.size == 0:
            break
        v[bad] = draw(bad.size)
    bad = u == v
    v[bad] = (u[bad] + 1) % n
    selfl = rng.random(S) < spec.p_self
    v[selfl] = u[selfl]
    start = rng.integers(0, spec.span, S, dtype=np.int64)
    k = rng.geometric(1.0 / spec.mu, S).astype(np.int64)

    total = int(k.sum())
    sess = np.repeat(np.arange(S, dtype=np.int64), k)
    first = np.zeros(total, bool)
    first[np.cumsum(k) - k] = True
    gap = rng.exponential(spec.beta, total)
    gap[first] = 0.0
    cg = np.cumsum(gap)
    base = cg[np.cumsum(k) - k]
    off = np.floor(cg - np.repeat(base, k)).astype(np.int64)
    t = start[sess] + off
    es = u[sess].copy()
    ed = v[sess].copy()
    rev = rng.random(total) < spec.p_reply
    es[rev], ed[rev] = ed[rev], es[rev].copy()

    if spec.fanout > 0:
        fo = rng.random(total) < spec.fanout
        idx = np.nonzero(fo)[0]
        extra = rng.integers(1, 5, idx.size)
        rep = np.repeat(idx, extra)
        xs = es[rep]
        xd = draw(rep.size)
        clash = xd == xs
        xd[clash] = (xs[clash] + 1) % n
        # interleave: each extra copy follows its parent event
        order_key = np.concatenate([np.arange(total, dtype=np.int64) * 8,
                                    rep * 8 + 1 + (np.arange(rep.size) - np.repeat(np.cumsum(extra) - extra, extra))])
        es = np.concatenate([es, xs]); ed = np.concatenate([ed, xd]); t = np.concatenate([t, t[rep]])
        o = np.argsort(order_key, kind="stable")
        es, ed, t = es[o], ed[o], t[o]

    keep = t < spec.span
    es, ed, t = es[keep], ed[keep], t[keep]
    if es.size < m:
        raise RuntimeError(f"generator produced {es.size} < {m} events; raise oversampling")
    es, ed, t = es[:m], ed[:m], t[:m]
    # (t, session, event): t < 2^33 and the session-order position < 2^30
    o = np.sort((t << 30) | np.arange(m, dtype=np.int64)) & ((1 << 30) - 1)
    src = es[o].astype(np.uint32)
    dst = ed[o].astype(np.uint32)
    tt = (t[o] + spec.t0).astype(np.int64)
    if shuffle:
        prm = np.random.default_rng(seed ^ 0x5EED).permutation(m)
        src, dst, tt = src[prm], dst[prm], tt[prm]
    return src, dst, tt, n


def config_graph(name: str, *, m: int | None = None, shuffle: bool = False, seed_offset: int = 0):
    idx = {"C1": 0, "C2": 1, "C3": 2, "C4": 3, "C5": 4}[name]
    return generate(SPECS[name], SEED_BASE + idx + seed_offset, m=m, shuffle=shuffle)


def tiny_graph(seed: int, n: int = 8, m: int = 40, tmax: int = 30, p_self: float = 0.05):
    """Small random multigraph for brute-force checks: many duplicate
    timestamps, parallel edges and some self-loops; input order random."""
    rng = np.random.default_rng(seed)
    src = rng.integers(0, n, m).astype(np.uint32)
    dst = rng.integers(0, n, m).astype(np.uint32)
    s = rng.random(m) < p_self
    dst[s] = src[s]
    t = rng.integers(0, tmax + 1, m).astype(np.int64)
    return src, dst, t, n


def burst_graph(seed: int, n: int = 2000, m_bg: int = 10000, span: int = 86400 * 7, bursts: int = 2,
                core: int = 48, burst_len: int = 600):
    """Skewed workload for the load-balancing row (§8 a8; "the top
    0.1% of the search trees constitute 34% of explored tree nodes"):
    a uniform random background plus `bursts` dense cores — `core` vertices
    exchanging every ordered pair once within `burst_len` seconds — so the
    few roots inside a core own almost all of the search work.  Input order
    random; timestamps integer seconds."""
    rng = np.random.default_rng(seed)
    src = [rng.integers(0, n, m_bg)]
    dst = [rng.integers(0, n, m_bg)]
    t = [rng.integers(0, span, m_bg)]
    for _ in range(bursts):
        vs = rng.choice(n, core, replace=False)
        a, b = np.meshgrid(vs, vs, indexing="ij")
        keep = a != b
        a, b = a[keep], b[keep]
        t0 = int(rng.integers(0, span - burst_len))
        src.append(a)
        dst.append(b)
        t.append(t0 + rng.integers(0, burst_len, a.shape[0]))
    src = np.concatenate(src).astype(np.uint32)
    dst = np.concatenate(dst).astype(np.uint32)
    t = np.concatenate(t).astype(np.int64)
    p = rng.permutation(src.shape[0])
    return src[p], dst[p], t[p], n


# ---------------------------------------------------------------- config C5
# Billion-edge eth-shaped graph (BASELINE.json configs[4]; SURVEY.md §8(d):
# n = 2^27, m ≈ 2e9, span 3.58 y, μ = 3.4, β = 10 min; α = 1.0, cap 0.3 %: calibrated
# with the oracle on a 1-day slice, to ~1e6 4-cycles per day
# against the eth dataset's 6.4e9 in 3.58 y).
# Too large to draw whole on one host, so it is generated in *time slices*:
# sessions are grouped into C5_BLOCKS blocks by start time, block b drawn
# from its own PCG64 stream (seed, b) and starting inside
# [b, b+1) · span / C5_BLOCKS.  A slice [ta, tb) draws only the blocks that
# can reach it (sessions last <= C5_MAX_SESSION s) and keeps the events in
# it, so every rank of a multi-GPU run draws exactly its own roots plus its
# δ-halo, and any two slices agree on the events they share.  Global order:
# (t, session, event).  m is ≈ 2e9 (the session count is fixed, events per
# session are random); vertex activity is the capped power law sampled in
# closed form: the top K ranks (share > cap) are drawn uniformly with mass
# K·cap, the rest by the inverse CDF of the continuous (r+1)^-α law, and
# ranks are scattered over the ids by the bijection r ↦ (r·φ32 + 12345) mod n.
C5 = GraphSpec("C5 billion-edge eth-shaped", 1 << 27, 2_000_000_000, int(3.58 * YEAR), 3.4, 1.0, 0.003, 600.0)
C5_BLOCKS = 8192
C5_MAX_SESSION = DAY
C5_MAX_EVENTS = 63


def _capped_zipf(rng, k, n, alpha, cap):
    # continuous (r+1)^-α law on ranks via G(x) = x^(1-α)/(1-α) (ln x at α = 1)
    if abs(alpha - 1.0) < 1e-12:
        G, Ginv = np.log, np.exp
    else:
        G = lambda x: np.power(x, 1.0 - alpha) / (1.0 - alpha)          # noqa: E731
        Ginv = lambda y: np.power(y * (1.0 - alpha), 1.0 / (1.0 - alpha))  # noqa: E731
    r = np.arange(1, 4097, dtype=np.float64)
    H = float(G(n + 0.5) - G(0.5))                                      # ≈ Σ_{r=1..n} r^-α
    K = int(((r ** -alpha) / H > cap).sum())
    head_mass = K * cap
    u = rng.random(k)
    head = u < head_mass
    out = np.empty(k, np.int64)
    if K:
        out[head] = np.minimum((u[head] / cap).astype(np.int64), K - 1)
    lo, hi = G(K + 0.5), G(n + 0.5)
    x = rng.random(int((~head).sum()))
    out[~head] = np.clip(np.floor(Ginv(lo + x * (hi - lo)) - 0.5), K, n - 1).astype(np.int64)
    return (out * 0x9E3779B1 + 12345) & (n - 1)    # n is a power of two: an odd multiplier permutes ids


def c5_block(b: int, seed: int = SEED_BASE + 4, spec: GraphSpec = C5):
    """Events of session block b: (t, session id, event index, src, dst),
    unsorted, t relative to the span start."""
    rng = np.random.default_rng([seed, b])
    S_total = int(math.ceil(spec.m / spec.mu))
    S = (S_total + C5_BLOCKS - 1) // C5_BLOCKS
    lo = b * spec.span // C5_BLOCKS
    hi = (b + 1) * spec.span // C5_BLOCKS
    u = _capped_zipf(rng, S, spec.n, spec.alpha, spec.cap)
    v = _capped_zipf(rng, S, spec.n, spec.alpha, spec.cap)
    clash = u == v
    v[clash] = (u[clash] + 1) & (spec.n - 1)
    selfl = rng.random(S) < spec.p_self
    v[selfl] = u[selfl]
    start = rng.integers(lo, hi, S, dtype=np.int64)
    k = np.minimum(rng.geometric(1.0 / spec.mu, S), C5_MAX_EVENTS).astype(np.int64)
    total = int(k.sum())
    sess = np.repeat(np.arange(S, dtype=np.int64), k)
    ev = np.arange(total, dtype=np.int64) - np.repeat(np.cumsum(k) - k, k)
    gap = rng.exponential(spec.beta, total)
    gap[ev == 0] = 0.0
    cg = np.cumsum(gap)
    off = np.floor(cg - np.repeat(cg[np.cumsum(k) - k], k)).astype(np.int64)
    t = start[sess] + off
    es, ed = u[sess], v[sess]
    rev = rng.random(total) < spec.p_reply
    es, ed = np.where(rev, ed, es), np.where(rev, es, ed)
    keep = (off <= C5_MAX_SESSION) & (t < spec.span)
    return t[keep], sess[keep] + b * S, ev[keep], es[keep], ed[keep]


def c5_slice(ta: int, tb: int, seed: int = SEED_BASE + 4, spec: GraphSpec = C5):
    """The C5 events with ta <= t < tb (relative seconds), ordered by
    (t, session, event): (src u32, dst u32, t i64 (absolute), n)."""
    b0 = max(0, (ta - C5_MAX_SESSION) * C5_BLOCKS // spec.span - 1)
    b1 = min(C5_BLOCKS, tb * C5_BLOCKS // spec.span + 1)
    keys, es, ds = [], [], []
    for b in range(b0, b1):
        t, sess, ev, s, d = c5_block(b, seed, spec)
        k = (t >= ta) & (t < tb)
        # (t, session, event) in one int64: t < 2^27 s, session < 2^30, event < 2^6
        keys.append((t[k] << 36) | (sess[k] << 6) | ev[k]); es.append(s[k].astype(np.uint32))
        ds.append(d[k].astype(np.uint32))
    key = np.concatenate(keys)
    o = np.argsort(key)
    return np.concatenate(es)[o], np.concatenate(ds)[o], (key[o] >> 36) + spec.t0, spec.n


def c5_rank_slice(rank: int, world: int, delta: int, seed: int = SEED_BASE + 4, spec: GraphSpec = C5):
    """Rank `rank` of `world`'s share of C5: the roots with t in an equal
    time range plus the forward δ-halo.  Returns (src, dst, t,
    n, n_roots): edges [0, n_roots) are the rank's roots."""
    ta = rank * spec.span // world
    tb = (rank + 1) * spec.span // world
    src, dst, t, n = c5_slice(ta, min(spec.span, tb + delta + 1), seed, spec)
    n_roots = int(np.searchsorted(t, tb + spec.t0, side="left"))
    return src, dst, t, n, n_roots
