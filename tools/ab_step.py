"""A/B timing of library variants on the bench step (one tm_count_multi over
the bench's motifs on config C4, L2 flushed between steps, CUDA events on the
library's stream).

    python tools/ab_step.py [--reps 7] [--motifs P3,TRI,C4,DIA] base variants/x/libtmotif.so ...

Each library runs in its own subprocess (TMOTIF_LIB); the graph is generated
once and cached in /tmp/tm_ab_<config>.npz for the duration of the call.  A
library named "base" is the in-tree build.  Prints one JSON line per library:
median step ms, per-kernel mine ms, the query-time passes (step - mining) and
the counts (which must agree across variants)."""
import argparse
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(a):
    import torch
    import bench
    from paper_2310_02800_b200 import tmotif as T
    bench.select_config(a.config)
    z = np.load(a.cache)
    src, dst, t, n = z["src"], z["dst"], z["t"], int(z["n"])
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    g = T.Graph(src, dst, t, n, device=0, stream=stream)
    names = a.motifs.split(",")
    mos = [T.Motif(*bench.motif_fine(x)[:1], bench.DELTA, bench.motif_fine(x)[1]) for x in names]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    steps, mines, cs = [], [], None
    for k in range(a.warmup + a.reps):
        with torch.cuda.stream(stream):
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        cs = T.tm_count_multi(g, mos, stream=stream, fuse=a.fuse)
        e1.record(stream)
        e1.synchronize()
        if k >= a.warmup:
            steps.append(e0.elapsed_time(e1))
            mines.append([x["mine_ms"] for x in T.tm_last_kernel_info()])
    i = int(np.argsort(steps)[len(steps) // 2])
    print(json.dumps({"lib": a.lib, "step_ms": steps[i], "min_step_ms": min(steps),
                      "mine_ms": dict(zip(names, [round(x, 3) for x in mines[i]])),
                      "passes_ms": round(steps[i] - sum(mines[i]), 3),
                      "counts": dict(zip(names, [int(c) for c in cs]))}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="*", default=["base"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--motifs", default="P3,TRI,C4,DIA")
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--fuse", type=int, default=0)
    ap.add_argument("--rounds", type=int, default=1, help="repeat the whole variant list (interleaved)")
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--lib", default="base")
    ap.add_argument("--cache", default="")
    a = ap.parse_args()
    if a.child:
        return child(a)
    cache = f"/tmp/tm_ab_{a.config}.npz"
    if not os.path.exists(cache):
        from paper_2310_02800_b200 import synth
        src, dst, t, n = synth.config_graph(a.config)
        np.savez(cache, src=src, dst=dst, t=t, n=n)
    for _ in range(a.rounds):
        for lib in a.libs:
            env = dict(os.environ)
            if lib != "base":
                env["TMOTIF_LIB"] = os.path.abspath(lib)
            subprocess.run([sys.executable, __file__, "--child", "--lib", lib, "--cache", cache, "--config", a.config,
                            "--motifs", a.motifs, "--reps", str(a.reps), "--warmup", str(a.warmup),
                            "--fuse", str(a.fuse)], env=env, check=False)


if __name__ == "__main__":
    main()
