"""Build the in-tree sm_100a shared library ``lib/libacp.so`` with nvcc.

Every CUDA source is compiled for ``-gencode arch=compute_100a,code=sm_100a``
with ``-lineinfo`` (ncu source view) and linked against the NCCL that
PyTorch ships (same soname, so one NCCL instance per process).
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "lib")
BUILD_DIR = os.path.join(OUT_DIR, "obj")
LIB_PATH = os.path.join(OUT_DIR, "libacp.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec and spec.submodule_search_locations:
        for base in spec.submodule_search_locations:
            cands.append(os.path.join(base, "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return os.path.join(c, "include"), os.path.join(c, "lib")
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def build_id() -> str:
    """Content hash of the library sources (csrc/ + include/acp.h): ties
    measurement artefacts (profiles/ncu_traffic_*.json) to the build they
    were captured on."""
    import hashlib
    h = hashlib.sha256()
    for f in sorted(glob.glob(os.path.join(CSRC, "*"))) + [os.path.join(ROOT, "include", "acp.h")]:
        if os.path.isfile(f):
            h.update(os.path.basename(f).encode())
            with open(f, "rb") as fh:
                h.update(fh.read())
    return h.hexdigest()[:16]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD_DIR, exist_ok=True)
    inc, libdir = _nccl_dirs()
    nvcc = _nvcc()
    headers = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "acp.h")]
    common = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
              "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc] + ARCH
    jobs = []
    objs = []
    for src in sources():
        obj = os.path.join(BUILD_DIR, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + headers):
            lang = ["-x", "cu"] if src.endswith(".cu") else []
            extra = ["-Xptxas", "-v"] if (verbose and src.endswith(".cu")) else []
            jobs.append([nvcc] + common + extra + lang + ["-c", src, "-o", obj])

    def run(cmd):
        p = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, p

    with cf.ThreadPoolExecutor(max_workers=min(8, max(1, os.cpu_count() or 1))) as ex:
        for cmd, p in ex.map(run, jobs):
            if verbose or p.returncode != 0:
                sys.stderr.write(" ".join(cmd) + "\n" + p.stdout + p.stderr)
            if p.returncode != 0:
                raise RuntimeError(f"nvcc failed for {cmd[-3]}")
    if force or jobs or _stale(LIB_PATH, objs):
        link = [nvcc, "-shared"] + ARCH + ["-o", LIB_PATH] + objs + \
            ["-L", libdir, "-l:libnccl.so.2", "-Xlinker", "-rpath," + libdir]
        p = subprocess.run(link, capture_output=True, text=True)
        if p.returncode != 0:
            sys.stderr.write(" ".join(link) + "\n" + p.stdout + p.stderr)
            raise RuntimeError("link failed")
    with open(os.path.join(OUT_DIR, "build_id.txt"), "w") as f:
        f.write(build_id() + "\n")
    return LIB_PATH


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
