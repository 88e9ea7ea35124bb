"""Builds libtmotif.so in-tree with nvcc for sm_100a (no JIT, no torch
extension machinery): every .cu under csrc/ is compiled in parallel and
linked into paper_2310_02800_b200/libtmotif.so."""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(CSRC, "build")
LIB = os.path.join(HERE, "libtmotif.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC,-O2",
         "-Xptxas", "-warn-spills"]


def _needs(obj, deps):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, jobs: int | None = None, extra_flags=(), lib: str = LIB, obj: str = OBJ) -> str:
    """extra_flags/lib/obj build a tuning variant (e.g. -DTM_MIN_BLOCKS=8) into another path."""
    global OBJ, LIB
    OBJ, LIB = obj, lib
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(HERE, "..", "include", "*.h"))
    objs = []
    todo = []
    for s in srcs:
        o = os.path.join(OBJ, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        if _needs(o, [s] + headers + [__file__]):
            todo.append((s, o))

    def comp(so):
        s, o = so
        cmd = [NVCC, *ARCH, *FLAGS, *extra_flags, "-c", s, "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {s}:\n{r.stderr}")
        return s, r.stderr

    jobs = jobs or min(8, os.cpu_count() or 1)
    with cf.ThreadPoolExecutor(jobs) as ex:
        for s, err in ex.map(comp, todo):
            if verbose:
                print("compiled", os.path.basename(s), file=sys.stderr)
                if err.strip():
                    print(err, file=sys.stderr)
    if todo or not os.path.exists(LIB):
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--variant", default=None, help="name of a tuning variant (built under variants/)")
    ap.add_argument("flags", nargs="*", help="extra nvcc flags, e.g. -DTM_MIN_BLOCKS=8")
    a = ap.parse_args()
    if a.variant:
        vd = os.path.join(HERE, "..", "variants", a.variant)
        print(build(verbose=True, extra_flags=a.flags, lib=os.path.join(vd, "libtmotif.so"), obj=os.path.join(vd, "obj")))
    else:
        print(build(verbose=True, extra_flags=a.flags))
