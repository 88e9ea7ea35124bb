#!/usr/bin/env python
"""Benchmark of the δ-temporal-motif hot path on B200 (BASELINE.json metric:
root edges/s and motif matches/s at 1/2/4/8 B200; % of HBM peak).

Workload (BASELINE.json config 4, the one the metric's 1/2/4/8-GPU scaling is
quoted on): stackoverflow-shaped synthetic temporal graph, n = 2,601,977,
m = 63,497,050 (Table 3), motifs P3, TRI, C4 (4-cycle), DIA
(5 edges) with δ = 1 day and a per-edge inter-event bound δ_i = 6 h on every
gap, counting.  One *step* = the four queries over every root edge, each
rebuilding its δ-horizons (query-time work) and running the mining kernel.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torchrun, one rank per GPU: ranks take contiguous,
work-balanced root ranges with their forward δ-halo (tm_partition_plan,
P:1020-1040), mine them with no inter-GPU traffic, and one NCCL all-reduce
combines the counts.  Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2310_02800_b200 import motifs as M  # noqa: E402
from paper_2310_02800_b200 import synth  # noqa: E402

# BASELINE.json configs the bench can run: C4 (default: the config the metric's
# 1/2/4/8-GPU scaling is quoted on) and C5 (the billion-edge one, drawn and
# mined in C5_PARTS time slices with δ-halos; rank r takes parts r, r+N, ...)
CONFIGS = {
    "C4": {"motifs": ["P3", "TRI", "C4", "DIA"], "delta": 86400, "fine": 21600, "index": 3},
    "C5": {"motifs": ["TRI", "C4"], "delta": 3600, "fine": None, "index": 4},
}
# 128 slices of ~15.6 M edges: per edge, smaller slices mine faster (their
# lists and pair filter stay closer to L2): a 1/8-slice's worth of roots took
# 1715 / 1449 / 1242 / 1108 / 1022 ms as 1 / 2 / 4 / 8 / 16 slices
# (profiles/r02_experiments.md); the forward δ-halo adds 0.4 % edges per slice
C5_PARTS = 128
CONFIG = "C4"
MOTIFS = CONFIGS[CONFIG]["motifs"]
DELTA = CONFIGS[CONFIG]["delta"]
FINE = CONFIGS[CONFIG]["fine"]


def select_config(name):
    global CONFIG, MOTIFS, DELTA, FINE
    CONFIG = name
    MOTIFS, DELTA, FINE = CONFIGS[name]["motifs"], CONFIGS[name]["delta"], CONFIGS[name]["fine"]
METRIC = "root edges/s"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
NCU_SUMMARY = os.path.join(ROOT, "profiles", "ncu_traffic.json")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def workload_config(world, m=None):
    spec = synth.C5 if CONFIG == "C5" else synth.SPECS[CONFIG]
    idx = CONFIGS[CONFIG]["index"]
    cfg = {"workload": f"{CONFIG} {spec.name.split(' ', 1)[1]} synthetic temporal graph (BASELINE.json configs[{idx}])",
           "n": spec.n, "m": m or spec.m, "motifs": MOTIFS, "delta_s": DELTA, "fine_delta_s": FINE,
           "mode": "count", "generator": {"alpha": spec.alpha, "cap": spec.cap, "mu": spec.mu, "beta_s": spec.beta,
                                          "seed": synth.SEED_BASE + idx},
           "partition": f"{world} contiguous root ranges + forward δ-halo" if world > 1 else "whole graph",
           "cache": "graph 2.3 GB > 126 MB L2; L2 flushed (256 MiB write) between timed steps"}
    if CONFIG == "C5":
        cfg["partition"] = (f"{C5_PARTS} equal time slices + forward δ-halo, rank r holds slices r, r+{world}, ...; "
                            f"each slice drawn, built and timed resident in turn")
        cfg["cache"] = "each slice's graph ~17 GB > 126 MB L2; L2 flushed (256 MiB write) between timed steps"
    return cfg


def pair_bucket_log2(t_sorted):
    """C5 graphs: edge-id buckets of the pair filter about two δ-windows wide
    (2^k >= 2 m δ / span), so a closing window covers at most two of them
    (C5 1/128 slice: k = 17, 66.2 -> 55.4 ms; profiles/r02_experiments.md)."""
    if CONFIG != "C5" or len(t_sorted) < 2:
        return 0
    span = max(1, int(t_sorted[-1]) - int(t_sorted[0]))
    per = 2.0 * len(t_sorted) * DELTA / span
    return max(1, int(math.ceil(math.log2(max(per, 2.0)))))


def motif_fine(name):
    mot = M.get(name)
    return mot, (None if FINE is None else [FINE] * (len(mot) - 1))


def balgo_bytes(stats, n_roots, L, fine=True):
    """Algorithmic bytes of one query, from the method's
    own instrumentation (tm_search_stats_run replays the oracle's Algorithm 1
    counters exactly: search nodes, Σ|window| under the shorter-list rule Q8):
      12 B per root            SRC[r], DST[r], H_δ[r]
      per internal search node  8 B  OFF[v], OFF[v+1]
                                4 B  H_δi[e_prev] (levels with a gap bound)
      8 B per candidate record in Algorithm 1's windows (window_sum).
    The §8(d) probe term (32 B x 2⌈log2(len+1)⌉ per node, the paper's two
    binary searches) is left out: this path resolves every window from a
    per-edge rank / window descriptor built once per query (k_hrank, its own
    kernel with its own bytes), so the dominant kernel performs no search; a
    literal probe term would exceed the HBM peak several times over
    (VERDICT r01 Weak #3)."""
    nodes = sum(stats["nodes"][1:L])
    return 12 * n_roots + (12 if fine else 8) * nodes + 8 * stats["window_sum"]


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, index):
        self.index = index
        self.lines = []
        self.p = None

    def resume(self):
        """Start sampling (the timed steps); pause() stops it for the untimed
        work in between (graph builds, the e2e pass: nvidia-smi's driver
        queries slow host-synchronous API sequences down)."""
        if self.p:
            return
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "50", "-i", str(self.index)], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, args=(self.p,), daemon=True)
            self.t.start()
        except OSError:
            self.p = None

    def pause(self):
        if self.p:
            time.sleep(0.25)
            self.p.terminate()
            self.p.wait()
            self.t.join(timeout=1.0)
            self.p = None

    def __enter__(self):
        return self

    def _read(self, proc):
        for line in proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        self.pause()

    def summary(self):
        sm, mx, reasons, under = [], 0.0, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                s, m_ = float(f[0]), float(f[1])
            except ValueError:
                continue
            sm.append(s)
            mx = max(mx, m_)
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
            under.append(s)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    try:
        d = json.load(open(PEAKS_PATH))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def peaks_field(key, default):
    try:
        return float(json.load(open(PEAKS_PATH))[key])
    except Exception:
        return default


# ------------------------------------------------------------------ oracle
def oracle_sample(src, dst, t, n, budget_s, seed=0, n_roots=None):
    """The oracle (Algorithm 1 in plain C, OpenMP over roots) as it stands,
    on all host cores, on a seeded uniform sample of roots of the same
    workload, sized to ~budget_s of CPU work.  Returns root edges/s etc."""
    import oracle
    threads = os.cpu_count() or 1
    og = oracle.Graph(src, dst, t, n)
    m = len(src) if n_roots is None else n_roots
    rng = np.random.default_rng(seed)
    k = 1 << 14
    spent, roots_done, matches, t_total = 0.0, 0, 0, 0.0
    while True:
        roots = np.sort(rng.choice(m, min(k, m), replace=False)).astype(np.uint64)
        t0 = time.perf_counter()
        for name in MOTIFS:
            mot, fine = motif_fine(name)
            matches += og.mine(mot, DELTA, fine, roots=roots, threads=threads)["count"]
        dt = time.perf_counter() - t0
        t_total += dt
        roots_done += len(roots) * len(MOTIFS)
        if t_total >= budget_s or k >= m:
            break
        k = int(min(m, k * max(2.0, min(8.0, (budget_s - t_total) / max(dt, 1e-3)))))
    return {"value": roots_done / t_total, "unit": "root edges/s", "cores": threads, "kind": "oracle",
            "sample": f"{roots_done // len(MOTIFS)} uniformly sampled roots (seeded) x {len(MOTIFS)} motifs of the "
                      f"{CONFIG} workload{' (time slice 0)' if CONFIG == 'C5' else ''}, {t_total:.1f} s on "
                      f"{threads} threads",
            "matches_per_s": matches / t_total}


def oracle_full(src, dst, t, n, counts):
    """Parity of the timed query's counts with the oracle over the WHOLE
    workload (every root, every motif; exact), run after the timed
    region on all host cores.  Its time is also the cpu_baseline: the oracle
    as it stands on the full workload."""
    import oracle
    threads = os.cpu_count() or 1
    og = oracle.Graph(src, dst, t, n)
    exp, t_total = [], 0.0
    for name in MOTIFS:
        mot, fine = motif_fine(name)
        t0 = time.perf_counter()
        exp.append(og.mine(mot, DELTA, fine, threads=threads)["count"])
        t_total += time.perf_counter() - t0
    m = len(src)
    return {"oracle_counts": dict(zip(MOTIFS, exp)), "match": [int(c) for c in counts] == exp,
            "oracle_s": t_total, "threads": threads, "scope": f"full workload: all {m} roots x {len(MOTIFS)} motifs",
            "cpu_baseline": {"value": m * len(MOTIFS) / t_total, "unit": "root edges/s", "cores": threads,
                             "kind": "oracle", "matches_per_s": sum(exp) / t_total,
                             "sample": f"the full {CONFIG} workload (all {m} roots x {len(MOTIFS)} motifs, "
                                       f"{t_total:.1f} s on {threads} threads); the same run is the parity check"}}


def run_reference(args):
    """--impl reference: the oracle on the host cores, same config/metric."""
    if CONFIG == "C5":
        src, dst, t, n, m = synth.c5_rank_slice(0, C5_PARTS, DELTA)
    else:
        src, dst, t, n = synth.config_graph(CONFIG)
        m = len(src)
    import oracle
    threads = os.cpu_count() or 1
    og = oracle.Graph(src, dst, t, n)
    per_step = 1 << 18
    rng = np.random.default_rng(1)

    def step():
        roots = np.sort(rng.choice(m, per_step, replace=False)).astype(np.uint64)
        c = 0
        for name in MOTIFS:
            mot, fine = motif_fine(name)
            c += og.mine(mot, DELTA, fine, roots=roots, threads=threads)["count"]
        return c

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    matches = 0
    for _ in range(args.steps):
        matches += step()
    dt = time.perf_counter() - t0
    roots = per_step * len(MOTIFS) * args.steps
    v = roots / dt
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "root edges/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1000 / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "i64",
            "data": "synthetic", "config": workload_config(args.gpus), "matches_per_s": matches / dt,
            "cpu_baseline": {"value": v, "unit": "root edges/s", "cores": threads, "kind": "oracle",
                             "sample": f"each step {per_step} uniformly sampled roots x {len(MOTIFS)} motifs"},
            "e2e": {"value": v, "unit": "root edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------------- ours
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true",
                    help="skip the full-workload oracle run (parity of the counts; also the cpu_baseline)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--config", choices=sorted(CONFIGS), default="C4")
    ap.add_argument("--separate", action="store_true",
                    help="one tm_count per motif instead of one tm_count_multi query (A/B)")
    args = ap.parse_args()
    select_config(args.config)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            run_reference(args)
        return
    args.warmup = max(args.warmup, 3)

    import torch
    import torch.distributed as dist
    from paper_2310_02800_b200 import multi
    from paper_2310_02800_b200 import tmotif as T

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    # ---- this rank's parts: (src, dst, t, n, root range); edges beyond the
    # root range are the forward δ-halo
    def parts():
        if CONFIG == "C5":
            for part in range(rank, C5_PARTS, world):
                t0 = time.time()
                s_, d_, t_, n_, nr = synth.c5_rank_slice(part, C5_PARTS, DELTA)
                log(f"[rank {rank}] C5 slice {part}/{C5_PARTS}: m={len(s_)} roots={nr} in {time.time() - t0:.1f}s")
                yield s_, d_, t_, n_, (0, nr)
            return
        t0 = time.time()
        src, dst, t, n = synth.config_graph(CONFIG)
        m = len(src)
        log(f"[rank {rank}] generated {CONFIG}: m={m} n={n} in {time.time() - t0:.1f}s")
        if world > 1:   # contiguous root ranges balanced by a per-root work proxy, + forward δ-halo
            reach = max(multi.reach(DELTA, motif_fine(x)[1]) for x in MOTIFS)
            w = multi.root_weights(src, dst, t, DELTA, FINE)
            a, b, e = multi.rank_slice(t, reach, world, rank, weights=w)
        else:
            a, b, e = 0, m, m
        yield tuple(np.ascontiguousarray(x[a:e]) for x in (src, dst, t)) + (n, (0, b - a))

    stream = torch.cuda.Stream(dev)
    motifs = [T.Motif(*motif_fine(name)[:1], DELTA, motif_fine(name)[1]) for name in MOTIFS]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    balance = [None] * len(MOTIFS)   # load balance of the last step's mining kernels (§8 a8)
    fused_into = [None] * len(MOTIFS)   # prefix fusion: the motif whose kernel counted this one
    kernel_mode = [0] * len(MOTIFS)     # tm_kernel_info.kernel_mode of the last step

    def step(g, rr):
        if args.separate:   # one tm_count per motif, each building its own horizons
            cs, mine, launches = [], [], 0
            for i, mo in enumerate(motifs):
                cs.append(T.tm_count(g, mo, root_range=rr, stream=stream))
                info = T.tm_last_run_info()
                mine.append(info["mine_ms"])
                launches += info["launches"]
                balance[i] = {"shared_tasks": info["shared_tasks"], "tail_ms": info["tail_ms"],
                              "warp_busy": info["warp_busy"]}
            return cs, mine, launches
        # one query for all motifs: the horizons / window-end ranks they share are built once
        cs = T.tm_count_multi(g, motifs, root_range=rr, stream=stream)
        kin = T.tm_last_kernel_info()
        for i, x in enumerate(kin):
            balance[i] = {"shared_tasks": x["shared_tasks"], "tail_ms": x["tail_ms"], "warp_busy": x["warp_busy"]}
            fused_into[i] = MOTIFS[x["carried_by"]] if x["carried_by"] >= 0 else None
            kernel_mode[i] = x["kernel_mode"]
        return cs, [x["mine_ms"] for x in kin], T.tm_last_run_info()["launches"]

    # ranks step together (per-step barrier + count all-reduce inside the timed
    # region) unless they hold different numbers of C5 slices
    lockstep = world > 1 and (CONFIG != "C5" or C5_PARTS % world == 0)

    def timed(fn):
        with torch.cuda.stream(stream):
            flush.zero_()                      # untimed L2 flush between steps
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        if lockstep:
            stream.synchronize()
            dist.barrier()                     # every rank starts the step together (§8(d))
        e0.record(stream)
        out = fn()
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1), out

    def reduced(fn):
        """fn's counts combined over the ranks inside the step: the one
        exchange of the multi-GPU path (NCCL all-reduce on the timed stream)."""
        def run():
            cs, mm, nl = fn()
            if lockstep:
                torch.cuda.nvtx.range_push("tm.allreduce_counts")
                with torch.cuda.stream(stream):
                    cs = multi.allreduce_counts(cs, device=dev)
                torch.cuda.nvtx.range_pop()
            return cs, mm, nl
        return run

    step_ms = np.zeros(args.steps)
    mine_ms = np.zeros(len(MOTIFS))
    counts = np.zeros(len(MOTIFS), np.int64)
    launches, my_roots, part0 = 0, 0, None
    e2e_ms, h2d = 0.0, 0
    nofuse_ms = 0.0
    with ClockSampler(local) as clk:
        for pi, (s_src, s_dst, s_t, n, rr) in enumerate(parts()):
            # C5 (coarse-only, hub-heavy): the pair index counts long closing windows (tm_graph_opts.pair_index)
            g = T.Graph(s_src, s_dst, s_t, n, device=local, stream=stream, pair_index=CONFIG == "C5",
                        pair_id_bucket_log2=pair_bucket_log2(s_t))
            for _ in range(args.warmup):
                step(g, rr)
            if lockstep:
                dist.barrier()
            torch.cuda.synchronize()
            clk.resume()
            for k in range(args.steps):
                ms, (cs, mm, nl) = timed(reduced(lambda: step(g, rr)))
                step_ms[k] += ms
                launches += nl
                if k == 0:
                    mine_ms += np.array(mm)
                    counts += np.array(cs, np.int64)   # already summed over the ranks
            clk.pause()
            if not args.separate:   # the same steps without prefix fusion, for transparency
                for _ in range(2):
                    T.tm_count_multi(g, motifs, root_range=rr, stream=stream, fuse=1)
                for k in range(args.steps):
                    nofuse_ms += timed(reduced(lambda: (T.tm_count_multi(g, motifs, root_range=rr, stream=stream,
                                                                           fuse=1), [], 0)))[0]
            my_roots += rr[1] - rr[0]
            if pi == 0:   # roofline inputs (untimed instrumentation runs) from this rank's first part
                stats = [T.tm_search_stats_run(g, mo, root_range=rr, stream=stream) for mo in motifs]
                part0 = {"roots": rr[1] - rr[0], "mine_ms": [None] * len(MOTIFS), "stats": stats,
                         "arrays": (s_src, s_dst, s_t, n, rr[1])}
                _, (_, mm0, _) = timed(lambda: step(g, rr))
                part0["mine_ms"] = mm0
                part0["balance"] = [dict(x) for x in balance]
                part0["fused_into"] = list(fused_into)
                part0["kernel_mode"] = list(kernel_mode)
            g.close()
            del g
            # ---- end to end through the public API from pinned host memory
            if not args.no_e2e:
                ph = [torch.from_numpy(x).pin_memory() for x in (s_src, s_dst, s_t)]
                hs, hd, ht = (x.numpy() for x in ph)

                def e2e_step():
                    gg = T.Graph(hs, hd, ht, n, device=local, stream=stream, pair_index=CONFIG == "C5",
                                 pair_id_bucket_log2=pair_bucket_log2(ht))
                    cs = ([T.tm_count(gg, mo, root_range=rr, stream=stream) for mo in motifs] if args.separate
                  else T.tm_count_multi(gg, motifs, root_range=rr, stream=stream))
                    gg.close()
                    return cs

                for _ in range(3):   # warm-up: grows the library's memory pool to a graph's size
                    e2e_step()
                torch.cuda.synchronize()
                e2e_each = []
                for _ in range(args.e2e_steps):
                    e2e_each.append(timed(reduced(lambda: (e2e_step(), [], 0)))[0])
                e2e_ms += sum(e2e_each)
                log(f"[rank {rank}] e2e steps (ms): " + " ".join(f"{x:.2f}" for x in e2e_each))
                h2d += int(sum(x.numel() * x.element_size() for x in ph))
                del ph, hs, hd, ht
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    total_ms = float(step_ms.sum())
    counts = [int(c) for c in counts]   # summed over the ranks inside every timed step
    if world > 1 and not lockstep:      # uneven C5 slice counts: combine once at the end
        counts = multi.allreduce_counts(counts, device=dev)
    tot = torch.tensor([total_ms, e2e_ms, nofuse_ms, float(my_roots), float(h2d)], dtype=torch.float64, device=dev)
    if world > 1:
        mx = tot[:3].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)   # max over ranks
        sm = tot[3:].clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        tot = torch.cat([mx, sm])
    total_ms, e2e_ms, nofuse_ms, all_roots, h2d_all = (float(x) for x in tot.tolist())
    roots_per_step = all_roots * len(MOTIFS)
    value = roots_per_step * args.steps / (total_ms / 1000)
    matches_per_s = sum(counts) * args.steps / (total_ms / 1000)

    # ---- roofline of the dominant kernel: algorithmic bytes per launch (the
    # method's own instrumentation on this rank's first part) ÷ its CUDA-event time
    bytes_q, per_motif = [], []
    for i, name in enumerate(MOTIFS):
        L = len(M.get(name))
        bq = balgo_bytes(part0["stats"][i], part0["roots"], L, fine=FINE is not None)
        bytes_q.append(bq)
        ms = part0["mine_ms"][i]
        fz = part0["fused_into"][i]
        resumed = part0.get("kernel_mode", [0] * len(MOTIFS))[i] == 5   # kResume: not a full search
        per_motif.append({"motif": name, "count": counts[i], "mine_ms": None if fz else ms,
                          "alg_bytes": bq, "alg_GBps": None if fz or resumed else bq / (ms / 1000) / 1e9,
                          "resumed_from_rows": resumed,
                          "search_nodes": sum(part0["stats"][i]["nodes"][1:L]),
                          "window_sum": part0["stats"][i]["window_sum"],
                          "load_balance": None if fz else part0["balance"][i],
                          "counted_inside": fz})
    dom = int(np.argmax(part0["mine_ms"]))

    def kernel_label(d, kmode, fused):
        name = {0: "kCount", 1: "kEnum", 4: "kCountPfx", 5: "kResume", 6: "kCountSib"}.get(kmode, str(kmode))
        inside = [MOTIFS[i] for i in range(len(MOTIFS)) if fused[i] == MOTIFS[d]]
        return f"mine_kernel<PlanC<{MOTIFS[d]}>, {name}>" + (f" (also counts {', '.join(inside)})" if inside else "")
    peak, peak_src = peaks()
    kmodes = part0.get("kernel_mode", [0] * len(MOTIFS))
    achieved = bytes_q[dom] / (part0["mine_ms"][dom] / 1000) / 1e9
    # ncu evidence of the same query (profiles/ncu_traffic.json, one `ncu --set
    # full` capture of every kernel of one step): DRAM bytes and executed warp
    # instructions per launch
    nc, dom_nc = None, None
    try:
        nc = json.load(open(NCU_SUMMARY))
        if nc.get("config") != CONFIG or world != 1:
            nc = None
        else:
            dom_nc = next((k for k in nc["kernels"] if k.get("motif") == MOTIFS[dom]), None)
    except Exception:
        nc = None
    props = torch.cuda.get_device_properties(dev)
    sm_max = peaks_field("sm_max_mhz", 1965.0)
    issue_peak = props.multi_processor_count * 4 * sm_max * 1e6 / 1e9   # G warp-instructions/s
    issue = None
    if dom_nc and dom_nc.get("warp_inst"):
        ia = dom_nc["warp_inst"] / (part0["mine_ms"][dom] / 1000) / 1e9
        issue = {"achieved": ia, "peak": issue_peak, "unit": "G warp-instructions/s", "frac": ia / issue_peak,
                 "warp_inst_per_launch": dom_nc["warp_inst"],
                 "peak_source": f"{props.multi_processor_count} SMs x 4 issue slots/clk x {sm_max:.0f} MHz "
                                f"(B200_PROFILING.md / MEASURED_PEAKS.json sm_max_mhz)"}
    hbm_alg = {"achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
               "bytes_per_launch": bytes_q[dom],
               "formula": "SURVEY 8(d) B_alg without the probe term: 12 m + 12 x search nodes + 8 x window_sum "
                          "(Algorithm 1's counters, shorter-list rule Q8)"}
    binding = "alu" if issue and issue["frac"] > hbm_alg["frac"] else "hbm"
    src_rl = issue if binding == "alu" else hbm_alg
    roofline = {"bound": binding, "achieved": src_rl["achieved"], "peak": src_rl["peak"], "unit": src_rl["unit"],
                "frac": src_rl["frac"], "traffic": dom_nc.get("dram_bytes") if dom_nc else None,
                "bound_note": "integer traversal: issue-bound when the issue fraction exceeds the algorithmic-HBM "
                              "fraction (both reported)",
                "issue": issue, "hbm_alg": hbm_alg,
                "kernel": kernel_label(dom, kmodes[dom], part0["fused_into"]),
                "peak_source": peak_src, "per_motif": per_motif,
                "ncu_source": NCU_SUMMARY.replace(ROOT + os.sep, "") if nc else None,
                "mine_share_of_step": float(mine_ms.sum() / (total_ms / args.steps))}
    hbm_pct = None
    if nc:   # ncu DRAM bytes over the query's kernels / T_query / peak
        q_dram = sum(k["dram_bytes"] for k in nc["kernels"])
        hbm_pct = q_dram / (total_ms / args.steps / 1000) / (peak * 1e9) * 100
        roofline["query_dram_bytes"] = q_dram
    e2e = None
    if not args.no_e2e:
        e2e = {"value": roots_per_step * args.e2e_steps / (e2e_ms / 1000), "unit": "root edges/s",
               "h2d_bytes_per_step": int(h2d_all), "d2h_bytes_per_step": 256 * len(MOTIFS) * world,
               "includes": f"graph load from pinned host (H2D + validate + sort + CSR build) + {len(MOTIFS)} "
                           f"queries + count read-back" + (f", for each of the {C5_PARTS} C5 slices"
                                                           if CONFIG == "C5" else "")}

    cpu, parity = None, None
    if rank == 0 and world == 1:   # after the timed region: the oracle on the host cores
        s_src, s_dst, s_t, n, nr = part0["arrays"]
        if CONFIG == "C4" and not args.no_parity:
            parity = oracle_full(s_src, s_dst, s_t, n, counts)
            cpu = parity.pop("cpu_baseline")
        elif not args.no_cpu_baseline:
            cpu = oracle_sample(s_src, s_dst, s_t, n, args.cpu_seconds, n_roots=nr)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "root edges/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
                "config": workload_config(world, int(all_roots) if CONFIG == "C5" else None),
                "matches_per_s": matches_per_s, "counts": dict(zip(MOTIFS, counts)),
                "hbm_pct_of_peak": hbm_pct, "roofline": roofline, "cpu_baseline": cpu, "parity": parity, "e2e": e2e,
                "clocks": clk.summary(), "gpu_launches": int(launches) * world,
                "gpu_launches_note": "per rank and step: 2 kernels per distinct horizon, one window-end-rank kernel per "
                                     "distinct (list, gap bound), one mining kernel per motif",
                "query": "one tm_count per motif" if args.separate else
                         "one tm_count_multi over the motifs (shared horizons and window descriptors; a motif "
                         "that is a prefix of another is counted as that motif's search-tree nodes)",
                "value_without_prefix_fusion": (roots_per_step * args.steps / (nofuse_ms / 1000)
                                                if nofuse_ms > 0 else None)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
