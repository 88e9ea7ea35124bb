"""Full-oracle parity and timing of every BASELINE.json config the oracle can
finish (SURVEY.md §8(d) "Oracle timing beside it": C1-C4 run the full oracle,
C1-C2 also single-threaded; C5 per-slice sampled roots).  For each config the
GPU runs the config's query (C1: TRI count + enumeration; C2: the 36-motif
census; C3: C4/TT/TT2 enumeration to a buffer sized by a prior count; C4: the
bench's fused P3/TRI/C4/DIA query with δ_i = 6 h; C5: one slice, TRI + C4)
and the oracle the same query over the same roots.  One JSON line per config:
counts, match, GPU ms (CUDA events of the library), oracle seconds and
threads.  usage: python tools/config_parity.py [C1 C2 ...]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2310_02800_b200 import motifs as M, synth, tmotif as T  # noqa: E402


def timed(fn):
    t0 = time.perf_counter()
    r = fn()
    return r, time.perf_counter() - t0


def run(cfg):
    out = {"config": cfg}
    if cfg == "C5":
        src, dst, t, n, nr = synth.c5_rank_slice(3, 8, 3600)
        out["slice"] = "3 of 8 (time range + δ-halo)"
    else:
        src, dst, t, n = synth.config_graph(cfg)
        nr = len(src)
    out.update(m=len(src), n=n, roots=nr)
    g = T.Graph(src, dst, t, n)
    og = oracle.Graph(src, dst, t, n)
    thr = oracle.max_threads()
    if cfg == "C1":
        mo = T.Motif(M.TRI, 3600)
        c = T.tm_count(g, mo)
        gms = T.tm_last_run_info()["total_ms"]
        rows, nt = T.tm_enumerate(g, mo, c, canonical=True)
        exp, osec = timed(lambda: og.mine(M.TRI, 3600, enumerate_=True, threads=thr))
        _, osec1 = timed(lambda: og.mine(M.TRI, 3600, threads=1))
        out.update(motifs=["TRI"], gpu=[c], oracle=[exp["count"]], gpu_ms=gms, oracle_s=osec, oracle_1thread_s=osec1,
                   rows_match=bool(np.array_equal(rows, exp["rows"])) and nt == exp["n_total"])
    elif cfg == "C2":
        got = [int(x) for x in T.tm_census36(g, 3600)]
        gms = T.tm_last_run_info()["total_ms"]
        exp, osec = timed(lambda: [og.mine(M.P36[k], 3600, threads=thr)["count"] for k in range(36)])
        _, osec1 = timed(lambda: [og.mine(M.P36[k], 3600, threads=1)["count"] for k in range(36)])
        out.update(motifs="P36 (all 36)", gpu=got, oracle=exp, gpu_ms=gms, oracle_s=osec, oracle_1thread_s=osec1)
    elif cfg == "C3":
        names = ["C4", "TT", "TT2"]
        got, gms, ok = [], 0.0, True
        exp, osec = timed(lambda: [og.mine(M.get(nm), 86400, threads=thr)["count"] for nm in names])
        for nm in names:
            mo = T.Motif(M.get(nm), 86400)
            c = T.tm_count(g, mo)
            rows, nt = T.tm_enumerate(g, mo, c)
            gms += T.tm_last_run_info()["total_ms"]
            got.append(c)
            ok = ok and nt == c
        out.update(motifs=names, gpu=got, oracle=exp, gpu_ms=gms, oracle_s=osec, enum_n_total_match=ok)
    elif cfg == "C4":
        spec = [("P3", [21600] * 2), ("TRI", [21600] * 2), ("C4", [21600] * 3), ("DIA", [21600] * 4)]
        got = T.tm_count_multi(g, [T.Motif(M.get(nm), 86400, f) for nm, f in spec])
        gms = T.tm_last_run_info()["total_ms"]
        exp, osec = timed(lambda: [og.mine(M.get(nm), 86400, f, threads=thr)["count"] for nm, f in spec])
        out.update(motifs=[nm for nm, _ in spec], gpu=got, oracle=exp, gpu_ms=gms, oracle_s=osec)
    else:   # C5: one slice, all its roots on the GPU; the oracle on 2^20 sampled roots (per-root counts)
        mos = [T.Motif(M.TRI, 3600), T.Motif(M.C4, 3600)]
        got = T.tm_count_multi(g, mos, root_range=(0, nr))
        gms = T.tm_last_run_info()["total_ms"]
        rng = np.random.default_rng(20)
        roots = np.sort(rng.choice(nr, 1 << 20, replace=False)).astype(np.uint64)
        gpu_s = [int(T.tm_count_roots(g, mo, roots).sum()) for mo in mos]
        exp, osec = timed(lambda: [int(og.mine(mm, 3600, roots=roots, per_root=True, threads=thr)["per_root"].sum())
                                   for mm in (M.TRI, M.C4)])
        out.update(motifs=["TRI", "C4"], gpu=got, gpu_ms=gms, sampled_roots=1 << 20, gpu_sampled=gpu_s,
                   oracle=exp, oracle_s=osec, note="oracle over 2^20 sampled roots vs per-root GPU counts")
        out["match"] = gpu_s == exp
    if "match" not in out:
        out["match"] = list(out["gpu"]) == list(out["oracle"])
    out["oracle_threads"] = thr
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    for c in (sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"]):
        run(c)
