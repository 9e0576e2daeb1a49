"""Build the in-tree CUDA library ``paper_2603_22300_b200/libsfa.so`` for sm_100a.

    python -m paper_2603_22300_b200.build [--force] [-v]

Every ``csrc/*.cu`` is compiled with nvcc (``-gencode arch=compute_100a,code=sm_100a -lineinfo
-O3``) into ``build/`` in parallel and linked into one shared library next to this file.
Incremental: a source is recompiled when it, or any ``csrc/*.cuh`` / ``include/*.h``, is newer
than its object; everything is rebuilt when the flags (incl. ``SFA_NVCC_FLAGS``) change.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import hashlib
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "libsfa.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", CSRC]


def extra_flags() -> list:
    """SFA_NVCC_FLAGS (space separated) is appended to every compile, e.g. -DSFA_WATCHDOG."""
    return os.environ.get("SFA_NVCC_FLAGS", "").split()


def nvcc() -> str:
    for c in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _deps_mtime() -> float:
    deps = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h"))
    return max((os.path.getmtime(p) for p in deps), default=0.0)


def _flags_stamp() -> str:
    """The compile configuration the objects in build/ were made with: a change of ARCH, FLAGS or
    SFA_NVCC_FLAGS (e.g. a -DSFA_WATCHDOG or -DSFA_MBAR_SUSPEND_NS=0 debug build) forces a full rebuild,
    so tests and the bench never link objects of another configuration."""
    return hashlib.sha256(" ".join(ARCH + FLAGS + extra_flags() + [nvcc()]).encode()).hexdigest()


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    stamp_path = os.path.join(BUILD, "flags.sha256")
    stamp = _flags_stamp()
    if not os.path.exists(stamp_path) or open(stamp_path).read().strip() != stamp:
        force = True
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    dep_t = _deps_mtime()
    objs, jobs = [], []
    for s in srcs:
        o = os.path.join(BUILD, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        if force or not os.path.exists(o) or os.path.getmtime(o) < max(os.path.getmtime(s), dep_t):
            cmd = [nvcc(), *ARCH, *FLAGS, *extra_flags(), "-c", s, "-o", o]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            jobs.append(cmd)
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
            for cmd, r in zip(jobs, ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), jobs)):
                if r.returncode != 0 or verbose:
                    sys.stderr.write(r.stdout + r.stderr)
                if r.returncode != 0:
                    raise RuntimeError(f"nvcc failed: {' '.join(cmd)}")
    if force or jobs or not os.path.exists(LIB):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call([nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-lcudart", "-ldl"])
        os.replace(tmp, LIB)
    with open(stamp_path, "w") as f:
        f.write(stamp + "\n")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
