"""Build libdgsip.so (the C-ABI of include/dg.h) in-tree with nvcc for sm_100a.

    python paper_2112_04167_b200/build.py [--pset 0x80] [--jobs N] [--force]

(run by path: importing the package itself requires the built library)

Every CUDA translation unit is compiled with
``-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo`` in parallel, then linked with
the static CUDA runtime.  NCCL is loaded at run time (dlopen) by multi-rank meshes only,
so only its header is needed here.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import hashlib
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INC = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libdgsip.so")
BUILD = os.path.join(HERE, "csrc", "build")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def nccl_include() -> str:
    try:
        import nvidia.nccl  # type: ignore

        base = os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0]
        inc = os.path.join(base, "include")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc
    except Exception:
        pass
    for c in glob.glob(os.path.join(sys.prefix, "lib", "python3*", "site-packages", "nvidia", "nccl", "include")):
        if os.path.exists(os.path.join(c, "nccl.h")):
            return c
    if os.path.exists("/usr/include/nccl.h"):
        return "/usr/include"
    raise RuntimeError("nccl.h not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                  [os.path.join(INC, "dg.h")])


def _digest(paths, extra=""):
    h = hashlib.sha1(extra.encode())
    for p in paths:
        with open(p, "rb") as f:
            h.update(f.read())
    return h.hexdigest()


def build(pset: str | None = None, jobs: int | None = None, force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    defs = [] if pset is None else ["-DDG_PSET=%s" % pset]
    defs += os.environ.get("DG_EXTRA_DEFS", "").split()  # development switches, e.g. -DDG_V5_DEBUG
    flags = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
             "-I" + INC, "-I" + CSRC, "-I" + nccl_include()] + defs
    hdr = _digest(headers(), " ".join(flags))
    stamp = os.path.join(BUILD, "stamp")
    want = _digest(sources(), hdr)
    if not force and not verbose and os.path.exists(LIB) and os.path.exists(stamp) and open(stamp).read() == want:
        return LIB

    def compile_one(src):
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        tag = obj + ".sha"
        key = _digest([src], hdr)
        if not force and os.path.exists(obj) and os.path.exists(tag) and open(tag).read() == key and \
                (not verbose or os.path.exists(obj + ".ptxas.log")):
            return obj
        cmd = [nvcc()] + ARCH + flags + ["-Xptxas", "-v"] * bool(verbose) + ["-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed for %s:\n%s\n%s" % (src, r.stdout, r.stderr))
        if verbose:
            with open(obj + ".ptxas.log", "w") as f:
                f.write(r.stderr)
        with open(tag, "w") as f:
            f.write(key)
        return obj

    srcs = sources()
    # the heavy template TUs first
    srcs.sort(key=lambda s: (0 if "apply" in s or "convect" in s else 1, s))
    with cf.ThreadPoolExecutor(max_workers=jobs or min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, srcs))
    tmp = LIB + ".tmp"
    cmd = [nvcc()] + ARCH + ["-shared", "-o", tmp] + objs + ["-ldl", "-lpthread"]
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    with open(stamp, "w") as f:
        f.write(want)
    return LIB


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pset", default=None, help="bit mask of compiled degrees (default: all)")
    ap.add_argument("--jobs", type=int, default=None)
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args()
    print(build(a.pset, a.jobs, a.force, a.verbose))


if __name__ == "__main__":
    main()
