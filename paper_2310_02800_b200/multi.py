"""Multi-GPU plumbing (§5.3).

Every search tree touches only edges in [r, H_δ(r)], so ranks
take contiguous, work-balanced root ranges and hold their roots plus a
forward δ-halo: no inter-GPU traffic while mining.  The one exchange is the
sum of the per-rank counts (torch.distributed all-reduce; NCCL on GPUs, gloo
in the CPU tests).  The split itself is the C-ABI's tm_partition_plan (host
code, no device needed).
"""
from __future__ import annotations

import numpy as np

from . import tmotif as T


def reach(delta: int, fine=None, anti=None) -> int:
    """How far past its root a search tree reads: the largest t(e_L) - t(e_1)
    of a match, min(δ, Σ δ_i), plus the longest anti-edge window (a witness
    may lie up to δ_ij after its attached edge)."""
    if fine is None or any(f is None or f >= T.DELTA_INF for f in fine):
        r = int(delta)
    else:
        r = int(min(delta, sum(int(f) for f in fine)))
    if anti:
        r += max(int(a[3]) for a in anti)
    return r


def root_weights(src_sorted, dst_sorted, t_sorted, delta: int, fine1=None):
    """Per-root work proxy for the split ("better: the
    level-2 window length"; the paper saw static splits by edge count plateau,
    P:1258): 1 + the number of edges leaving dst(r) in (r, H(r)], H the
    tighter of δ and the first gap bound δ_1 — the candidate window of the
    motif edge 1 -> 2 that every bench motif starts with, whose size sets how
    many level-2 subtrees root r spawns.  Host numpy, sorted edge order."""
    S = np.asarray(src_sorted, np.int64)
    D = np.asarray(dst_sorted, np.int64)
    t = np.asarray(t_sorted, np.int64)
    m = len(t)
    ids = np.arange(m, dtype=np.int64)
    d = int(delta) if fine1 is None else min(int(delta), int(fine1))
    H = np.searchsorted(t, t + d, side="right") - 1          # last id within the window
    key = np.sort(S << 32 | ids)                              # out-lists: (source, id) in order
    lo = np.searchsorted(key, D << 32 | ids, side="right")
    hi = np.searchsorted(key, D << 32 | H, side="right")
    return (1 + hi - lo).astype(np.uint64)


def rank_slice(t_sorted, reach_s: int, world: int, rank: int, weights=None):
    """(root_lo, root_hi, edge_hi) of `rank`: it mines roots [root_lo, root_hi)
    on the sorted edges [root_lo, edge_hi) (its roots + forward halo)."""
    lo, hi = T.tm_partition_plan(np.ascontiguousarray(t_sorted, np.int64), reach_s, world, weights)
    return int(lo[rank]), int(lo[rank + 1]), int(hi[rank])


def allreduce_counts(counts, device=None):
    """Sum per-rank count vectors over the default process group (int64)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([int(c) for c in counts], dtype=torch.int64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [int(x) for x in t.tolist()]
