"""CPU-only checks of the C ABI: the library loads, exports every symbol
include/tmotif.h declares, and its host-side logic (motif validation and
canonicalisation, the partition planner) behaves — no kernel is launched."""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2310_02800_b200 import tmotif as T

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tmotif.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tm_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = T.lib()
    names = declared_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    # the binding wraps exactly the declared set
    assert sorted(n for n, _, _ in T.SIGNATURES) == names


def test_version_and_no_error():
    assert "sm_100a" in T.tm_version()


def test_motif_validation_and_specialisation():
    # catalog motifs get compile-time specialised kernels, whatever their labels
    assert T.Motif([(0, 1), (1, 2), (2, 0)], 3600).specialised
    assert T.Motif([(7, 3), (3, 9), (9, 7)], 3600).specialised          # relabelled TRI
    assert T.Motif([(0, 1), (1, 2), (2, 3), (3, 0)], 10).specialised    # C4
    assert not T.Motif([(0, 1), (1, 0), (1, 2), (2, 1)], 10).specialised  # generic runtime plan
    # prefix-disconnected (Q9): accepted, searched by the thread-per-root kernel, not specialisable
    mo = T.Motif([(0, 1), (2, 3)], 10)
    assert not mo.specialised
    with pytest.raises(T.TMotifError) as e:
        mo.specialise()
    assert e.value.status == T.TM_EUNSUPPORTED
    for bad in ([(0, 0)], [], [(0, 1)] * 7, [(0, 64)]):
        with pytest.raises(T.TMotifError) as e:
            T.Motif(bad, 10)
        assert e.value.status == T.TM_EINVAL
    with pytest.raises(T.TMotifError):
        T.Motif([(0, 1)], -1)
    with pytest.raises(T.TMotifError):
        T.Motif([(0, 1), (1, 2)], 5, [-3])
    # 7 vertices allowed, 8 not
    T.Motif([(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 6)], 5)


def test_graph_create_rejects_bad_input_without_gpu():
    # host-side validation fails before any device work
    for s, d, t, n in (([0], [5], [0], 2), ([0], [1], [-1], 2)):
        with pytest.raises(T.TMotifError) as e:
            T.Graph(np.array(s), np.array(d), np.array(t), n)
        assert e.value.status == T.TM_EINVAL


def test_partition_plan_tiles_roots_and_covers_halo():
    rng = np.random.default_rng(0)
    t = np.sort(rng.integers(0, 10_000, 5000)).astype(np.int64)
    for P in (1, 2, 3, 8):
        for delta in (0, 50, 700):
            lo, hi = T.tm_partition_plan(t, delta, P)
            assert lo[0] == 0 and lo[-1] == len(t)
            assert np.all(np.diff(lo.astype(np.int64)) >= 0)
            for p in range(P):
                if lo[p + 1] > lo[p]:
                    last = int(lo[p + 1]) - 1
                    # one past the last edge within δ of the last root
                    assert hi[p] == np.searchsorted(t, t[last] + delta, side="right")
    # balanced by the default proxy (window length)
    lo, _ = T.tm_partition_plan(t, 100, 4)
    w = np.searchsorted(t, t + 100, side="right") - np.arange(len(t))
    parts = [w[int(lo[p]):int(lo[p + 1])].sum() for p in range(4)]
    assert max(parts) < 1.1 * (sum(parts) / 4) + w.max()
    with pytest.raises(T.TMotifError):
        T.tm_partition_plan(t[::-1], 10, 2)


def test_declared_struct_sizes_match_binding():
    # the ctypes mirrors must match the C layout (x86-64 SysV)
    # stream, root_lo/hi/offset, canonical, on_device, grid, block, share, fuse
    assert ctypes.sizeof(T.RunOpts) == 8 + 8 * 3 + 4 * 2 + 4 * 2 + 4 + 4
    assert T.RunOpts.share.offset == 48 and T.RunOpts.fuse.offset == 52
    # 3 f32 + 3 u32, shared_tasks u64, tail_ms, warp_busy
    assert ctypes.sizeof(T.RunInfo) == 24 + 8 + 4 + 4
    assert T.RunInfo.shared_tasks.offset == 24
    assert ctypes.sizeof(T.KernelInfo) == 32 and T.KernelInfo.shared_tasks.offset == 16
    assert T.KernelInfo.carried_by.offset == 24
    assert T.KernelInfo.kernel_mode.offset == 28
    assert ctypes.sizeof(T.SearchStats) == 8 * 13
    # device, (pad), stream, input_on_device, pair_index, pair_id_bucket_log2, (pad)
    assert ctypes.sizeof(T.GraphOpts) == 32
    assert T.GraphOpts.stream.offset == 8 and T.GraphOpts.pair_id_bucket_log2.offset == 24


def test_kernel_mode_constants_match_header():
    import re
    txt = open(HEADER).read()
    want = {m.group(1): int(m.group(2)) for m in re.finditer(r"#define TM_KMODE_(\w+)\s+\(?(-?\d+)\)?", txt)}
    assert want == {"NONE": -1, "COUNT": 0, "ENUM": 1, "COUNT_PREFIX": 4, "RESUME": 5, "COUNT_SIB": 6, "DFS": 7}
    for k, v in want.items():
        assert getattr(T, "KMODE_" + k) == v
