"""In-tree build of the native libraries (no JIT cache: the .so files travel
with the repo snapshot to the GPU box).

  libmprec_gpu.so  -- the product: sm_100a kernels + C++ host runtime (nvcc)
  libmprec_gen.so  -- synthetic input generator (g++)
  oracle/liboracle.so -- the CPU checker (g++, test infrastructure)
  oracle/_ref/libmprec_ref.so -- the reference's own sources + Eigen shim (checker pin)
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX", "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _run(cmd, cwd=None):
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=cwd)


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_gen(force=False):
    src = os.path.join(CSRC, "gen", "mprec_gen.cpp")
    out = os.path.join(HERE, "libmprec_gen.so")
    deps = [src, os.path.join(CSRC, "gen", "mprec_gen.h")]
    if force or _stale(out, deps):
        _run([CXX, "-O2", "-std=c++17", "-fPIC", "-shared", "-ffp-contract=off", "-pthread", "-o", out, src])
    return out


REFERENCE_SRC = "/root/reference/proj/src"


def build_oracle(force=False):
    """oracle/liboracle.so (the restatement) and, where the reference tree is
    present (this container; never the GPU box), oracle/_ref/libmprec_ref.so:
    the reference's own sources compiled against the Eigen-subset shim.
    Building the checker is not using it: only tests/, smoke() and bench.py's
    reference arm load these."""
    odir = os.path.join(ROOT, "oracle")
    _run(["make", "-s", "-C", odir] + (["-B"] if force else []))
    if os.path.isdir(REFERENCE_SRC):
        _run(["make", "-s", "-C", odir, "ref"] + (["-B"] if force else []))
    return os.path.join(odir, "liboracle.so")


def gpu_sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def build_gpu(force=False, checked=False):
    """libmprec_gpu.so, or with checked=True libmprec_gpu_checked.so: the same
    sources with -DMPREC_CHECKED (device-side bounds checks in the sync-free and
    level-synchronous kernels, MG_DCHECK) -- test infrastructure standing in for
    compute-sanitizer, which this GPU pool does not allow."""
    out = os.path.join(HERE, "libmprec_gpu_checked.so" if checked else "libmprec_gpu.so")
    srcs = gpu_sources()
    hdrs = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + [
        os.path.join(ROOT, "include", "mprec_gpu.h")]
    if not srcs:
        return None
    if not (force or _stale(out, srcs + hdrs)):
        return out
    objdir = os.path.join(HERE, "_obj_checked" if checked else "_obj")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"),
                    "-I", CSRC, "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]
    if checked:
        flags += ["-DMPREC_CHECKED"]
    for s in srcs:
        o = os.path.join(objdir, os.path.basename(s) + ".o")
        if force or _stale(o, [s] + hdrs):
            # *_exact.cu hold the setup kernels that must be bitwise equal to the
            # oracle: no FMA contraction there.
            extra = ["-fmad=false"] if s.endswith("_exact.cu") else []
            _run([NVCC] + flags + extra + ["-c", s, "-o", o])
        objs.append(o)
    _run([NVCC] + ARCH + ["-shared", "-o", out] + objs + ["-lcudart"])
    return out


def build_all(force=False):
    build_gen(force)
    build_gpu(force)
    build_gpu(force, checked=True)
    if os.path.exists(os.path.join(ROOT, "oracle", "Makefile")):
        build_oracle(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
