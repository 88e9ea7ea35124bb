"""Thin ctypes binding of libtmotif.so (C ABI in include/tmotif.h).

Argument marshalling only: every step of the path runs in the library's CUDA
kernels.  Functions keep the C names (``tm_graph_create``, ``tm_count`` ...);
``Graph``/``Motif`` are small RAII wrappers around the handles.  Buffers may
be numpy arrays (host) or torch CUDA tensors (device; PyTorch supplies device
memory and streams only).  There is no CPU fallback: if the library is
missing this module raises on first use.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# TMOTIF_LIB selects a tuning variant of the same library (variants/<name>/libtmotif.so)
LIB_PATH = os.environ.get("TMOTIF_LIB") or os.path.join(_HERE, "libtmotif.so")

TM_OK, TM_EINVAL, TM_ENOMEM, TM_ECUDA, TM_EUNSUPPORTED, TM_TRUNCATED = range(6)
DELTA_INF = (1 << 63) - 1
MAX_EDGES = 6
_STATUS = {1: "TM_EINVAL", 2: "TM_ENOMEM", 3: "TM_ECUDA", 4: "TM_EUNSUPPORTED", 5: "TM_TRUNCATED"}

_P = ctypes.c_void_p
_u64, _u32, _i64, _i32, _f32 = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int64, ctypes.c_int, ctypes.c_float


class TMotifError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class GraphOpts(ctypes.Structure):
    _fields_ = [("device", _i32), ("stream", _P), ("input_on_device", _i32), ("pair_index", _i32),
                ("pair_id_bucket_log2", _i32)]


class RunOpts(ctypes.Structure):
    _fields_ = [("stream", _P), ("root_lo", _u64), ("root_hi", _u64), ("edge_id_offset", _u64),
                ("canonical", _i32), ("buffers_on_device", _i32), ("grid_ctas", _u32),
                ("block_threads", _u32), ("share", _i32), ("fuse", _i32)]


class SearchStats(ctypes.Structure):
    _fields_ = [("nodes", _u64 * 8), ("window_sum", _u64), ("list_sum", _u64), ("probe_sum", _u64),
                ("matches", _u64), ("fast_window_sum", _u64)]


class RunInfo(ctypes.Structure):
    _fields_ = [("horizon_ms", _f32), ("mine_ms", _f32), ("total_ms", _f32), ("launches", _u32),
                ("grid_ctas", _u32), ("block_threads", _u32), ("shared_tasks", _u64),
                ("tail_ms", _f32), ("warp_busy", _f32)]


# tm_kernel_info.kernel_mode (tmotif.h TM_KMODE_*)
KMODE_NONE, KMODE_COUNT, KMODE_ENUM, KMODE_COUNT_PREFIX, KMODE_RESUME, KMODE_COUNT_SIB, KMODE_DFS = -1, 0, 1, 4, 5, 6, 7


class KernelInfo(ctypes.Structure):
    _fields_ = [("mine_ms", _f32), ("tail_ms", _f32), ("warp_busy", _f32), ("grid_ctas", _u32),
                ("shared_tasks", _u64), ("carried_by", _i32), ("kernel_mode", _i32)]


_lib = None
_lock = threading.Lock()

# (name, restype, argtypes) of every symbol include/tmotif.h declares
SIGNATURES = [
    ("tm_graph_create", _i32, [_P, _P, _P, _u64, _u32, ctypes.POINTER(GraphOpts), ctypes.POINTER(_P)]),
    ("tm_graph_destroy", _i32, [_P]),
    ("tm_graph_info", _i32, [_P, ctypes.POINTER(_u64), ctypes.POINTER(_u32), ctypes.POINTER(_i32)]),
    ("tm_graph_sorted_to_input", _i32, [_P, _P]),
    ("tm_graph_sorted_edges", _i32, [_P, _P, _P, _P]),
    ("tm_motif_create", _i32, [_u32, _P, _P, _i64, _P, ctypes.POINTER(_P)]),
    ("tm_motif_destroy", _i32, [_P]),
    ("tm_graph_set_labels", _i32, [_P, _P, _P, _i32]),
    ("tm_motif_set_vertex_label", _i32, [_P, _u32, _i32]),
    ("tm_motif_set_edge_label", _i32, [_P, _u32, _i32]),
    ("tm_motif_add_anti_edge", _i32, [_P, _u32, _u32, _u32, _i64]),
    ("tm_motif_specialised", _i32, [_P, ctypes.POINTER(_i32)]),
    ("tm_motif_specialise", _i32, [_P]),
    ("tm_run_opts_default", None, [ctypes.POINTER(RunOpts)]),
    ("tm_count", _i32, [_P, _P, ctypes.POINTER(RunOpts), ctypes.POINTER(_u64)]),
    ("tm_enumerate", _i32, [_P, _P, ctypes.POINTER(RunOpts), _P, _u64, ctypes.POINTER(_u64),
                            ctypes.POINTER(_u64)]),
    ("tm_count_roots", _i32, [_P, _P, ctypes.POINTER(RunOpts), _P, _u64, _P]),
    ("tm_search_stats_run", _i32, [_P, _P, ctypes.POINTER(RunOpts), ctypes.POINTER(SearchStats)]),
    ("tm_census36", _i32, [_P, _i64, _P, ctypes.POINTER(RunOpts), _P]),
    ("tm_count_multi", _i32, [_P, _P, _u32, ctypes.POINTER(RunOpts), _P]),
    ("tm_last_kernel_info", _i32, [ctypes.POINTER(KernelInfo), _u32, ctypes.POINTER(_u32)]),
    ("tm_last_run_info", _i32, [ctypes.POINTER(RunInfo)]),
    ("tm_partition_plan", _i32, [_P, _u64, _i64, _u32, _P, _P, _P]),
    ("tm_last_error", ctypes.c_char_p, []),
    ("tm_version", ctypes.c_char_p, []),
]


def lib():
    """Load libtmotif.so (raises if it was not built — no fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} missing: build it with `python -c 'import __graft_entry__ as g; "
                                  f"g.build()'` (there is no CPU fallback)")
            L = ctypes.CDLL(LIB_PATH)
            for name, res, args in SIGNATURES:
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib


def _check(st: int):
    if st != TM_OK:
        raise TMotifError(st, lib().tm_last_error().decode())


def _is_torch(a):
    return type(a).__module__.startswith("torch")


def _host_ptr(a):
    return a.ctypes.data_as(_P)


def _ptr(a):
    """Pointer of a numpy array (host) or a torch tensor (its data_ptr())."""
    if a is None:
        return None
    if _is_torch(a):
        return _P(a.data_ptr())
    return _host_ptr(a)


def _stream_handle(stream):
    if stream is None:
        return None
    if isinstance(stream, int):
        return _P(stream)
    return _P(stream.cuda_stream)  # torch.cuda.Stream


def run_opts(stream=None, root_range=None, edge_id_offset=0, canonical=False, buffers_on_device=False,
             grid_ctas=0, share=0, fuse=0) -> RunOpts:
    """share: heavy-subtree sharing, 0 on (default), 1 off, 2 eager; fuse: prefix
    fusion in tm_count_multi, 0 on (default), 1 off (tm_run_opts)."""
    o = RunOpts()
    lib().tm_run_opts_default(ctypes.byref(o))
    o.stream = _stream_handle(stream)
    if root_range is not None:
        o.root_lo, o.root_hi = int(root_range[0]), int(root_range[1])
    o.edge_id_offset = int(edge_id_offset)
    o.canonical = int(bool(canonical))
    o.buffers_on_device = int(bool(buffers_on_device))
    o.grid_ctas = int(grid_ctas)
    o.share = int(share)
    o.fuse = int(fuse)
    return o


# ----------------------------------------------------------------- handles
class Graph:
    """tm_graph: device-resident sorted edge list + bidirectional CSR."""

    def __init__(self, src, dst, t, n_vertices: int, *, device: int = -1, stream=None, pair_index: bool = False,
                 pair_id_bucket_log2: int = 0):
        L = lib()
        on_dev = _is_torch(src)
        if on_dev:
            import torch
            src = src.to(torch.int32).contiguous()
            dst = dst.to(torch.int32).contiguous()
            t = t.to(torch.int64).contiguous()
            if device < 0:
                device = src.device.index
        else:
            src = np.ascontiguousarray(src, np.uint32)
            dst = np.ascontiguousarray(dst, np.uint32)
            t = np.ascontiguousarray(t, np.int64)
        self._keep = (src, dst, t)
        m = int(src.shape[0])
        o = GraphOpts(device, _stream_handle(stream), int(on_dev), int(bool(pair_index)), int(pair_id_bucket_log2))
        h = _P()
        _check(L.tm_graph_create(_ptr(src), _ptr(dst), _ptr(t), m, int(n_vertices), ctypes.byref(o),
                                 ctypes.byref(h)))
        self._keep = None
        self._h = h
        mm, nn, dd = _u64(), _u32(), _i32()
        _check(L.tm_graph_info(h, ctypes.byref(mm), ctypes.byref(nn), ctypes.byref(dd)))
        self.m, self.n, self.device = int(mm.value), int(nn.value), int(dd.value)

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.tm_graph_destroy(self._h)
        self._h = None

    __del__ = close

    def set_labels(self, vlabels=None, elabels=None):
        """Vertex labels (n) and edge labels (m, the caller's input order);
        numpy / host or torch CUDA int32 tensors; None leaves that kind at 0."""
        on_dev = _is_torch(vlabels) or _is_torch(elabels)
        conv = []
        for x, k in ((vlabels, self.n), (elabels, self.m)):
            if x is None:
                conv.append(None)
                continue
            if on_dev:
                import torch
                x = x.to(torch.int32).contiguous()
            else:
                x = np.ascontiguousarray(x, np.int32)
            if int(x.shape[0]) != k:
                raise ValueError("label array length")
            conv.append(x)
        _check(lib().tm_graph_set_labels(self._h, None if conv[0] is None else _ptr(conv[0]),
                                         None if conv[1] is None else _ptr(conv[1]), int(on_dev)))

    def sorted_to_input(self) -> np.ndarray:
        perm = np.empty(self.m, np.uint64)
        _check(lib().tm_graph_sorted_to_input(self._h, _host_ptr(perm)))
        return perm

    def sorted_edges(self):
        s = np.empty(self.m, np.uint32); d = np.empty(self.m, np.uint32); t = np.empty(self.m, np.int64)
        _check(lib().tm_graph_sorted_edges(self._h, _host_ptr(s), _host_ptr(d), _host_ptr(t)))
        return s, d, t


class Motif:
    """tm_motif: ordered motif edges + δ + optional per-gap δ_i."""

    def __init__(self, edges, delta: int, fine=None, *, vlabels=None, elabels=None, anti=None):
        """vlabels: {motif vertex: label}; elabels: per motif edge label or
        None; anti: [(u, v, attach, window)] (generalized query)."""
        L = len(edges)
        mu = np.array([int(e[0]) for e in edges], np.uint32)
        mv = np.array([int(e[1]) for e in edges], np.uint32)
        fa = None
        if fine is not None:
            fa = np.array([DELTA_INF if f is None else int(f) for f in fine], np.int64)
            if fa.shape[0] != max(L - 1, 0):
                raise ValueError("fine needs L-1 entries")
        h = _P()
        _check(lib().tm_motif_create(L, _host_ptr(mu), _host_ptr(mv), int(delta),
                                     None if fa is None else _host_ptr(fa), ctypes.byref(h)))
        self._h = h
        for v, lab in (vlabels or {}).items():
            _check(lib().tm_motif_set_vertex_label(h, int(v), int(lab)))
        for i, lab in enumerate(elabels or []):
            if lab is not None:
                _check(lib().tm_motif_set_edge_label(h, i, int(lab)))
        for (u, v, a, w) in (anti or []):
            _check(lib().tm_motif_add_anti_edge(h, int(u), int(v), int(a), int(w)))
        self.L = L
        self.edges = [tuple(e) for e in edges]
        self.delta = delta
        self.fine = fine

    @property
    def handle(self):
        return self._h

    @property
    def specialised(self) -> bool:
        s = _i32()
        _check(lib().tm_motif_specialised(self._h, ctypes.byref(s)))
        return bool(s.value)

    def specialise(self):
        """Compile this motif's own kernels with NVRTC (tm_motif_specialise)."""
        _check(lib().tm_motif_specialise(self._h))
        return self

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.tm_motif_destroy(self._h)
        self._h = None

    __del__ = close


# -------------------------------------------------------------- the calls
def tm_count(g: Graph, mo: Motif, **opts) -> int:
    c = _u64()
    o = run_opts(**opts)
    _check(lib().tm_count(g.handle, mo.handle, ctypes.byref(o), ctypes.byref(c)))
    return int(c.value)


def tm_enumerate(g: Graph, mo: Motif, cap: int, buf=None, **opts):
    """Returns (rows, n_total).  buf: None (host numpy result), a numpy
    (cap, L) uint32 array, or a torch CUDA int32 tensor (written in place)."""
    on_dev = buf is not None and _is_torch(buf)
    if buf is None:
        buf = np.zeros((max(cap, 1), mo.L), np.uint32)
    elif on_dev:
        import torch
        if buf.dtype not in (torch.int32, torch.uint32) or not buf.is_contiguous() or buf.numel() < cap * mo.L:
            raise ValueError("device buffer must be a contiguous int32 tensor of at least (cap, L) elements")
    else:
        if buf.dtype != np.uint32 or not buf.flags.c_contiguous or buf.size < cap * mo.L:
            raise ValueError("host buffer must be a C-contiguous uint32 array of at least (cap, L) elements")
    o = run_opts(buffers_on_device=on_dev, **opts)
    nt, nw = _u64(), _u64()
    st = lib().tm_enumerate(g.handle, mo.handle, ctypes.byref(o), _ptr(buf), int(cap), ctypes.byref(nt),
                            ctypes.byref(nw))
    if st not in (TM_OK, TM_TRUNCATED):
        _check(st)
    return buf[: int(nw.value)], int(nt.value)


def tm_count_roots(g: Graph, mo: Motif, roots, **opts):
    if _is_torch(roots):
        import torch
        # the C side reads u64 ids and does not range-check device buffers
        roots = roots.to(torch.int64).contiguous().reshape(-1)
        if roots.numel() and (int(roots.min()) < 0 or int(roots.max()) >= g.m):
            raise ValueError("root id out of range [0, m)")
        counts = torch.zeros(roots.shape[0], dtype=torch.int64, device=roots.device)
        o = run_opts(buffers_on_device=True, **opts)
    else:
        roots = np.ascontiguousarray(roots, np.uint64)
        counts = np.zeros(roots.shape[0], np.uint64)
        o = run_opts(**opts)
    _check(lib().tm_count_roots(g.handle, mo.handle, ctypes.byref(o), _ptr(roots), int(roots.shape[0]),
                                _ptr(counts)))
    return counts


def tm_search_stats_run(g: Graph, mo: Motif, **opts) -> dict:
    s = SearchStats()
    o = run_opts(**opts)
    _check(lib().tm_search_stats_run(g.handle, mo.handle, ctypes.byref(o), ctypes.byref(s)))
    return {"nodes": list(s.nodes), "window_sum": s.window_sum, "list_sum": s.list_sum,
            "probe_sum": s.probe_sum, "matches": s.matches, "fast_window_sum": s.fast_window_sum}


def tm_count_multi(g: Graph, motifs, **opts) -> list:
    """Counts of several motifs in one query (shared horizons / window-end ranks)."""
    k = len(motifs)
    arr = (_P * k)(*[mo.handle for mo in motifs])
    counts = np.zeros(k, np.uint64)
    o = run_opts(**opts)
    _check(lib().tm_count_multi(g.handle, arr, k, ctypes.byref(o), _host_ptr(counts)))
    return [int(c) for c in counts]


def tm_last_kernel_info() -> list:
    n = _u32()
    _check(lib().tm_last_kernel_info(None, 0, ctypes.byref(n)))
    buf = (KernelInfo * max(1, n.value))()
    _check(lib().tm_last_kernel_info(buf, n.value, ctypes.byref(n)))
    return [{"mine_ms": b.mine_ms, "tail_ms": b.tail_ms, "warp_busy": b.warp_busy, "grid_ctas": b.grid_ctas,
             "shared_tasks": b.shared_tasks, "carried_by": b.carried_by,
             "kernel_mode": b.kernel_mode} for b in buf[: n.value]]


def tm_census36(g: Graph, delta: int, fine=None, **opts) -> np.ndarray:
    """36 counts, index a*6+b = motif (0→1, E6[a], E6[b]) (motifs.P36 order)."""
    counts = np.zeros(36, np.uint64)
    fa = None
    if fine is not None:
        fa = np.array([DELTA_INF if f is None else int(f) for f in fine], np.int64)
        if fa.shape[0] != 2:
            raise ValueError("fine needs 2 entries")
    o = run_opts(**opts)
    _check(lib().tm_census36(g.handle, int(delta), None if fa is None else _host_ptr(fa), ctypes.byref(o),
                             _host_ptr(counts)))
    return counts


def tm_last_run_info() -> dict:
    r = RunInfo()
    _check(lib().tm_last_run_info(ctypes.byref(r)))
    return {"horizon_ms": r.horizon_ms, "mine_ms": r.mine_ms, "total_ms": r.total_ms, "launches": r.launches,
            "grid_ctas": r.grid_ctas, "block_threads": r.block_threads, "shared_tasks": r.shared_tasks,
            "tail_ms": r.tail_ms, "warp_busy": r.warp_busy}


def tm_partition_plan(t_sorted, delta: int, P: int, weights=None):
    t_sorted = np.ascontiguousarray(t_sorted, np.int64)
    w = None if weights is None else np.ascontiguousarray(weights, np.uint64)
    lo = np.zeros(P + 1, np.uint64)
    hi = np.zeros(P, np.uint64)
    _check(lib().tm_partition_plan(_host_ptr(t_sorted), int(t_sorted.shape[0]), int(delta), int(P),
                                   None if w is None else _host_ptr(w), _host_ptr(lo), _host_ptr(hi)))
    return lo, hi


def tm_version() -> str:
    return lib().tm_version().decode()
