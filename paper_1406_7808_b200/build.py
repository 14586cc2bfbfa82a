"""Build the SR-FMG shared library in-tree with nvcc for sm_100a (B200).

    python paper_1406_7808_b200/build.py          # incremental
    python paper_1406_7808_b200/build.py --force

Produces paper_1406_7808_b200/libsrfmg.so (C ABI of include/sr_fmg.h).  No GPU needed:
nvcc cross-compiles.  Static CUDA runtime; no torch headers or symbols.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(HERE, "libsrfmg.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["kernels.cu", "fused.cu", "fused27.cu", "prolong.cu", "pset.cu", "up.cu", "restrict.cu", "coarse.cu", "solver.cpp"]
HEADERS = ["kernels.cuh", "fused.cuh", "tma.cuh", "coarse.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3", "-I", CSRC,
         "-I", os.path.join(ROOT, "include"), "--expt-relaxed-constexpr"]


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else -1.0


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = [s for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    hdr_t = max([_mtime(os.path.join(CSRC, h)) for h in HEADERS] +
                [_mtime(os.path.join(ROOT, "include", "sr_fmg.h")), _mtime(__file__)])
    objs, jobs = [], []
    for s in srcs:
        src = os.path.join(CSRC, s)
        obj = os.path.join(BUILD, s + ".o")
        objs.append(obj)
        if force or _mtime(obj) < max(_mtime(src), hdr_t):
            cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
            if s.endswith(".cu"):
                cmd += ["-Xptxas", "-v"] if verbose else []
            else:
                cmd += ["-x", "cu"]
            jobs.append((s, cmd))
    # the translation units are independent: compile them concurrently
    from concurrent.futures import ThreadPoolExecutor
    workers = max(1, min(len(jobs), os.cpu_count() or 1))
    with ThreadPoolExecutor(max_workers=workers) as ex:
        results = list(ex.map(lambda j: (j[0], subprocess.run(j[1], capture_output=True, text=True)),
                              jobs))
    for s, r in results:
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {s}")
        if verbose:
            sys.stderr.write(r.stderr)
    if force or _mtime(LIB) < max(_mtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-Xcompiler", "-fPIC"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc link failed")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
