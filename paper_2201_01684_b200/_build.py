"""Build libgpoeo.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

The .so is git-ignored but travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libgpoeo.so")
SOURCES = ["gpoeo_api.cu", "composite.cu", "spectrum.cu", "score.cu", "select.cu", "rolling.cu", "gear.cu"]
HEADERS = ["gpoeo_internal.cuh"]
EXTRA = os.environ.get("GPOEO_NVCC_EXTRA", "").split()
NVCC_FLAGS = EXTRA + ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(INCLUDE, "gpoeo.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None, extra: list | None = None) -> str:
    """Build libgpoeo.so (or, with out/extra, a variant with extra nvcc flags at `out`: the
    profiling experiments' builds, loaded through GPOEO_LIB)."""
    if out is None and not force and not _stale():
        return LIB
    lib = out or LIB
    flags = NVCC_FLAGS + (extra or [])
    objs = []
    procs = []
    for src in SOURCES:
        obj = lib + "." + src.replace(".cu", ".o")
        cmd = ["nvcc", *flags, "-I", INCLUDE, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append(subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
        objs.append(obj)
    for p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out)
            raise RuntimeError("nvcc failed")
        if verbose and out:
            sys.stderr.write(out)
    tmp = lib + ".tmp"
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs])
    os.replace(tmp, lib)
    for o in objs:
        os.remove(o)
    return lib


if __name__ == "__main__":
    # python _build.py [--force] [-v] [--out PATH -- extra nvcc flags...]
    argv = sys.argv[1:]
    extra = argv[argv.index("--") + 1:] if "--" in argv else []
    out = argv[argv.index("--out") + 1] if "--out" in argv else None
    print(build(force="--force" in argv, verbose="-v" in argv, out=out, extra=extra))
