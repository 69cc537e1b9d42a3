"""Build libsnk.so in-tree: nvcc for sm_100a only (no other arch, no JIT).

    python -m paper_1804_06304_b200.build [--verbose] [--force]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
# SNK_BUILD_TAG (tuning experiments only): objects and library under a tagged name
_TAG = os.environ.get("SNK_BUILD_TAG", "")
OBJ = os.path.join(HERE, "build_obj" + (f"_{_TAG}" if _TAG else ""))
LIB = os.path.join(HERE, f"libsnk_{_TAG}.so" if _TAG else "libsnk.so")
SOURCES = ["abi.cu", "volume.cu", "stencil.cu", "seeds.cu", "evolve.cu", "cull.cu", "label.cu"]
HEADERS = ["common.cuh", "tma.cuh"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
BASE = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off",
        "-I", os.path.join(ROOT, "include"), "--expt-relaxed-constexpr"]
# evolve.cu: every FMA is explicit, so no contraction can differ between schedules
PER_FILE = {"evolve.cu": ["-fmad=false"]}


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _stale(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    deps = [src, os.path.join(ROOT, "include", "snk.h")] + [os.path.join(CSRC, h) for h in HEADERS]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    cc = nvcc()
    jobs = []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(OBJ, s.replace(".cu", ".o"))
        if force or _stale(obj, src):
            # SNK_NVCC_EXTRA: extra -D flags for tuning experiments (scripts/)
            extra = os.environ.get("SNK_NVCC_EXTRA", "").split()
            cmd = [cc, *ARCH, *BASE, *PER_FILE.get(s, []), *extra, "-c", src, "-o", obj]
            if verbose:
                cmd += ["-Xptxas", "-v"]
            jobs.append((s, cmd))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        futs = {ex.submit(subprocess.run, cmd, capture_output=True, text=True): s for s, cmd in jobs}
        errors = []
        for f in cf.as_completed(futs):
            r = f.result()
            if verbose or r.returncode != 0:
                sys.stderr.write(f"--- {futs[f]}\n{r.stdout}{r.stderr}")
            if r.returncode != 0:
                errors.append(futs[f])
        if errors:
            raise RuntimeError(f"nvcc failed for {errors}")
    objs = [os.path.join(OBJ, s.replace(".cu", ".o")) for s in SOURCES]
    if force or jobs or not os.path.exists(LIB):
        tmp = LIB + ".tmp"
        subprocess.check_call([cc, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"])
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose))
