"""In-tree build of the sm_100a kernels into ``_lib/libtcb200.so`` (nvcc, no torch JIT).

Used by ``__graft_entry__.build()`` and ``python -m paper_2505_16864_b200._build``.
Objects are rebuilt only when a source or header is newer than the object.
"""

from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "_lib")
OBJ_DIR = os.path.join(OUT_DIR, "obj")
LIB = os.path.join(OUT_DIR, "libtcb200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
    "-Xptxas", "-v", "-I", os.path.join(ROOT, "include"),
] + os.environ.get("TCB_NVCC_EXTRA", "").split()  # e.g. -DTCB_CARVE_TRACE for timeline builds


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _deps_mtime() -> float:
    files = glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "tokencarve_b200.h")]
    return max(os.path.getmtime(f) for f in files)


def _flags_changed() -> bool:
    stamp = os.path.join(OBJ_DIR, "flags.txt")
    cur = " ".join(NVCC_FLAGS)
    old = open(stamp).read() if os.path.exists(stamp) else None
    return old != cur


def _compile(src: str, verbose: bool, force: bool = False) -> str:
    obj = os.path.join(OBJ_DIR, os.path.basename(src).replace(".cu", ".o"))
    if (not force and os.path.exists(obj)
            and os.path.getmtime(obj) >= max(os.path.getmtime(src), _deps_mtime())):
        return obj
    cmd = [nvcc(), *NVCC_FLAGS, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    log = os.path.join(OBJ_DIR, os.path.basename(src) + ".ptxas.txt")
    with open(log, "w") as fh:
        fh.write(r.stderr)
    if verbose:
        sys.stderr.write(r.stderr)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ_DIR, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    force = _flags_changed()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, force), srcs))
    with open(os.path.join(OBJ_DIR, "flags.txt"), "w") as fh:
        fh.write(" ".join(NVCC_FLAGS))
    if force and os.path.exists(LIB):
        os.remove(LIB)
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", LIB, *objs, "-lcuda" if False else "-lcudart_static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
