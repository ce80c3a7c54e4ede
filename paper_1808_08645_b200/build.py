"""Build libbbwadg.so in-tree for sm_100a (nvcc, parallel, mtime-incremental).

    python -m paper_1808_08645_b200.build [--clean] [-j 8]

Output: paper_1808_08645_b200/native/libbbwadg.so (git-ignored, travels to the GPU
box with the gpurun snapshot).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
# BBWADG_VARIANT=<name> + BBWADG_DEFS="-DBBW_T=128 ..." build a tuning variant into native/<name>/
VARIANT = os.environ.get("BBWADG_VARIANT", "")
EXTRA_DEFS = os.environ.get("BBWADG_DEFS", "").split()
if EXTRA_DEFS and not VARIANT:
    # tuning defines must not leak into (or hide inside) the production library
    raise SystemExit("BBWADG_DEFS needs BBWADG_VARIANT=<name> (builds into native/<name>/)")
BUILD = os.path.join(HERE, "build", VARIANT) if VARIANT else os.path.join(HERE, "build")
LIBDIR = os.path.join(HERE, "native", VARIANT) if VARIANT else os.path.join(HERE, "native")
LIB = os.path.join(LIBDIR, "libbbwadg.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "-Xcompiler", "-fopenmp",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _headers_mtime():
    hs = glob.glob(os.path.join(CSRC, "*.hpp")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "bbwadg.h")]
    return max(os.path.getmtime(h) for h in hs)


def _defs_stamp_changed() -> bool:
    """A variant rebuilt with different BBWADG_DEFS must recompile every object."""
    stamp = os.path.join(BUILD, "defs.txt")
    want = " ".join(EXTRA_DEFS)
    have = open(stamp).read() if os.path.exists(stamp) else None
    if have != want:
        with open(stamp, "w") as fh:
            fh.write(want)
        return True
    return False


def _compile(src: str, hdr_mtime: float, verbose: bool, force: bool = False) -> str:
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_mtime):
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, *EXTRA_DEFS, "-c", src, "-o", obj]
    if src.endswith(".cpp"):
        cmd = [NVCC, "-x", "cu", *ARCH, *FLAGS, *EXTRA_DEFS, "-c", src, "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {os.path.basename(src)}:\n{r.stderr[-6000:]}")
    if verbose and r.stderr:
        with open(obj + ".ptxas.txt", "w") as fh:
            fh.write(r.stderr)
    return obj


def build(jobs: int | None = None, clean: bool = False, verbose: bool = False) -> str:
    if clean and os.path.isdir(BUILD):
        shutil.rmtree(BUILD)
    os.makedirs(BUILD, exist_ok=True)
    os.makedirs(LIBDIR, exist_ok=True)
    hm = _headers_mtime()
    srcs = _sources()
    force = _defs_stamp_changed()
    jobs = jobs or min(len(srcs), os.cpu_count() or 4)
    with cf.ThreadPoolExecutor(jobs) as ex:
        objs = list(ex.map(lambda s: _compile(s, hm, verbose, force), srcs))
    if os.path.exists(LIB) and os.path.getmtime(LIB) >= max(os.path.getmtime(o) for o in objs):
        return LIB
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart", "-ldl", "-lgomp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--clean", action="store_true")
    ap.add_argument("-j", type=int, default=None)
    ap.add_argument("-v", action="store_true", help="keep ptxas -v reports next to the objects")
    a = ap.parse_args()
    print(build(a.j, a.clean, a.v))
    sys.exit(0)
