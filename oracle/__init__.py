"""oracle — TEST INFRASTRUCTURE ONLY (not product code).

Python handle on ``oracle/tmoracle.c``, the plain CPU implementation of the
paper's Algorithm 1 that every CUDA result is checked
against.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package.  It shares
no code with ``paper_2310_02800_b200`` and never imports it.

The library is compiled with plain ``gcc -O2 -fopenmp`` on first use (or by
``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tmoracle.c")
_LIB = os.path.join(_HERE, "libtmoracle.so")
_lock = threading.Lock()
_lib = None

INF = (1 << 63) - 1  # δ = ∞
MAXL = 8
MAXV = 16
MAXANTI = 4
ANY = -1             # no label requirement

OK, EINVAL, ENOMEM, EUNSUPPORTED = 0, 1, 2, 3
_ERRS = {EINVAL: "invalid argument", ENOMEM: "out of memory", EUNSUPPORTED: "unsupported motif (prefix-disconnected, Q9)"}


class OracleError(RuntimeError):
    def __init__(self, code: int):
        super().__init__(f"oracle status {code}: {_ERRS.get(code, '?')}")
        self.code = code


class Stats(ctypes.Structure):
    """Instrumentation of Algorithm 1 (see tmoracle.c header)."""
    _fields_ = [("nodes", ctypes.c_uint64 * MAXL), ("window_sum", ctypes.c_uint64),
                ("list_sum", ctypes.c_uint64), ("probe_sum", ctypes.c_uint64),
                ("matches", ctypes.c_uint64)]

    def as_dict(self):
        return {"nodes": list(self.nodes), "window_sum": self.window_sum, "list_sum": self.list_sum,
                "probe_sum": self.probe_sum, "matches": self.matches}


class Constraints(ctypes.Structure):
    """Labels / anti-edges of the generalized query (tmo_constraints)."""
    _fields_ = [("vlabel", ctypes.c_int32 * MAXV), ("elabel", ctypes.c_int32 * MAXL), ("n_anti", ctypes.c_uint32),
                ("anti_u", ctypes.c_uint32 * MAXANTI), ("anti_v", ctypes.c_uint32 * MAXANTI),
                ("anti_attach", ctypes.c_uint32 * MAXANTI), ("anti_window", ctypes.c_int64 * MAXANTI)]


def make_constraints(vlabels=None, elabels=None, anti=None):
    """vlabels: {motif vertex: label}; elabels: per motif edge label or None;
    anti: [(u, v, attach, window)] — attach = 0-based real motif edge."""
    if not vlabels and not elabels and not anti:
        return None
    c = Constraints()
    for i in range(MAXV):
        c.vlabel[i] = ANY
    for i in range(MAXL):
        c.elabel[i] = ANY
    for v, lab in (vlabels or {}).items():
        c.vlabel[int(v)] = int(lab)
    for i, lab in enumerate(elabels or []):
        if lab is not None:
            c.elabel[i] = int(lab)
    anti = list(anti or [])
    if len(anti) > MAXANTI:
        raise ValueError("too many anti-edges")
    c.n_anti = len(anti)
    for j, (u, v, a, w) in enumerate(anti):
        c.anti_u[j], c.anti_v[j], c.anti_attach[j], c.anti_window[j] = int(u), int(v), int(a), int(w)
    return c


def build(force: bool = False) -> str:
    """Compile tmoracle.c -> libtmoracle.so (plain gcc, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared", "-Wall",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            u64, u32, i64, i32 = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int64, ctypes.c_int
            lib.tmo_graph_build.argtypes = [P, P, P, u64, u32, ctypes.POINTER(P)]
            lib.tmo_graph_build.restype = i32
            lib.tmo_graph_free.argtypes = [P]
            lib.tmo_graph_free.restype = None
            lib.tmo_graph_export.argtypes = [P, P, P, P, P]
            lib.tmo_graph_export.restype = None
            lib.tmo_mine.argtypes = [P, u32, P, P, i64, P, P, u64, u64, P, u64, i32, P, P, P, u64, P, P]
            lib.tmo_graph_set_labels.argtypes = [P, P, P]
            lib.tmo_graph_set_labels.restype = i32
            lib.tmo_mine.restype = i32
            lib.tmo_max_threads.argtypes = []
            lib.tmo_max_threads.restype = i32
            _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def max_threads() -> int:
    return int(_load().tmo_max_threads())


class Graph:
    """Chronologically sorted temporal edge list + in/out CSR."""

    def __init__(self, src, dst, t, n_vertices: int):
        lib = _load()
        self._src = np.ascontiguousarray(src, dtype=np.uint32)
        self._dst = np.ascontiguousarray(dst, dtype=np.uint32)
        self._t = np.ascontiguousarray(t, dtype=np.int64)
        self.m = int(self._src.shape[0])
        self.n = int(n_vertices)
        h = ctypes.c_void_p()
        rc = lib.tmo_graph_build(_ptr(self._src), _ptr(self._dst), _ptr(self._t), self.m, self.n,
                                 ctypes.byref(h))
        if rc:
            raise OracleError(rc)
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.tmo_graph_free(h)
            self._h = None

    def set_labels(self, vlabels=None, elabels=None):
        """Vertex labels (n) and edge labels (m, input order); None = all 0."""
        va = None if vlabels is None else np.ascontiguousarray(vlabels, np.int32)
        ea = None if elabels is None else np.ascontiguousarray(elabels, np.int32)
        if va is not None and va.shape[0] != self.n or ea is not None and ea.shape[0] != self.m:
            raise ValueError("label array length")
        rc = _load().tmo_graph_set_labels(self._h, _ptr(va), _ptr(ea))
        if rc:
            raise OracleError(rc)
        self._labels = (va, ea)

    def sorted_arrays(self):
        """(perm, src, dst, t) in sorted edge-id order; perm[id] = input position."""
        m = self.m
        perm = np.empty(m, np.uint64); s = np.empty(m, np.uint32); d = np.empty(m, np.uint32)
        t = np.empty(m, np.int64)
        _load().tmo_graph_export(self._h, _ptr(perm), _ptr(s), _ptr(d), _ptr(t))
        return perm, s, d, t

    def mine(self, motif, delta: int, fine=None, *, root_range=None, roots=None, threads: int = 0,
             per_root: bool = False, enumerate_: bool = False, cap: int | None = None,
             vlabels=None, elabels=None, anti=None):
        """Run Algorithm 1.  Returns dict(count, stats, per_root?, rows?, n_total?).
        vlabels / elabels / anti: the generalized query's constraints
        (make_constraints)."""
        cons = make_constraints(vlabels, elabels, anti)
        lib = _load()
        L = len(motif)
        mu = np.array([e[0] for e in motif], np.uint32)
        mv = np.array([e[1] for e in motif], np.uint32)
        fa = None
        if fine is not None:
            fa = np.array([INF if f is None else int(f) for f in fine], np.int64)
            if fa.shape[0] != L - 1:
                raise ValueError("fine must have L-1 entries")
        lo, hi = (0, self.m) if root_range is None else root_range
        ra = None if roots is None else np.ascontiguousarray(roots, np.uint64)
        nr = 0 if ra is None else int(ra.shape[0])
        n_iter = nr if ra is not None else max(0, min(hi, self.m) - lo)
        pr = np.zeros(n_iter, np.uint64) if per_root else None
        buf, ntot = None, None
        if enumerate_:
            if cap is None:
                cap = int(self.mine(motif, delta, fine, root_range=root_range, roots=roots,
                                    threads=threads, vlabels=vlabels, elabels=elabels, anti=anti)["count"])
            buf = np.zeros((max(cap, 1), L), np.uint32)
            ntot = np.zeros(1, np.uint64)
        cnt = np.zeros(1, np.uint64)
        st = Stats()
        rc = lib.tmo_mine(self._h, L, _ptr(mu), _ptr(mv), int(delta), _ptr(fa),
                          None if cons is None else ctypes.byref(cons), int(lo), int(hi),
                          _ptr(ra), nr, int(threads), _ptr(cnt), _ptr(pr), _ptr(buf),
                          int(cap or 0), _ptr(ntot), ctypes.byref(st))
        if rc:
            raise OracleError(rc)
        out = {"count": int(cnt[0]), "stats": st.as_dict()}
        if per_root:
            out["per_root"] = pr
        if enumerate_:
            n_total = int(ntot[0])
            out["n_total"] = n_total
            out["rows"] = buf[:min(n_total, cap)]
        return out


def count(src, dst, t, n, motif, delta, fine=None, threads=0):
    """Convenience: build + count."""
    return Graph(src, dst, t, n).mine(motif, delta, fine, threads=threads)["count"]
