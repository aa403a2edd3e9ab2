"""Build libnlse_b200.so in-tree with nvcc for sm_100a.

The library is several translation units (csrc/nlse_api.cu + one inst_*.cu per kernel
family), compiled to objects in parallel and linked with `nvcc -shared`.

Flags that matter for the result: -fmad=false (no FMA
contraction), IEEE division / no FTZ (nvcc defaults, no --use_fast_math).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
import time
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libnlse_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false", "-prec-div=true", "-ftz=false",
    "-Xcompiler", "-fPIC,-O2",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sorted(glob.glob(os.path.join(CSRC, "*")) + [os.path.join(ROOT, "include", "nlse.h")])


def up_to_date(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return False
    t = os.path.getmtime(lib)
    return all(os.path.getmtime(d) <= t for d in deps())


def build_to(lib: str, defines=(), log: str | None = None, jobs: int | None = None) -> str:
    """Compile every translation unit with the extra -D `defines` and link `lib`."""
    objdir = os.path.join(os.path.dirname(lib), "build", os.path.splitext(os.path.basename(lib))[0])
    os.makedirs(objdir, exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include")]

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        cmd = [NVCC, *NVCC_FLAGS, *defines, *inc, "-c", "-o", obj, src]
        t0 = time.time()
        r = subprocess.run(cmd, capture_output=True, text=True)
        r.stdout += f"\n[build] {os.path.basename(src)}: {time.time() - t0:.1f} s\n"
        return obj, cmd, r

    jobs = jobs or max(1, min(len(sources()), os.cpu_count() or 1))
    with ThreadPoolExecutor(jobs) as ex:
        results = list(ex.map(compile_one, sources()))
    text, failed = [], False
    for obj, cmd, r in results:
        text.append(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        failed |= r.returncode != 0
    tmp = lib + f".tmp{os.getpid()}"
    if not failed:
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp,
               *[o for o, _, _ in results], "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        text.append(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        failed = r.returncode != 0
    if log:
        with open(log, "w") as fh:
            fh.write("\n".join(text))
    if failed:
        sys.stderr.write("\n".join(t for t in text if "error" in t)[-20000:])
        raise RuntimeError(f"nvcc failed (see {log})")
    os.replace(tmp, lib)
    return lib


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    log = os.path.join(HERE, "build_ptxas.log")
    build_to(LIB, log=log)
    if verbose:
        sys.stderr.write(open(log).read())
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
