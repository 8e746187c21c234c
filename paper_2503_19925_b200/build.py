"""Build the in-tree shared libraries for sm_100a with nvcc.

  libpoly.so       the product: C ABI of include/poly.h (K1..K4 kernels)
  libpolysynth.so  CUDA twin of gen/rng.py (input generation only; -fmad=false)

Both link the CUDA runtime statically so the .so files load on a CPU-only
box (ABI/symbol tests) and on the GPU box without a JIT cache.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O2", "-shared",
          "--cudart", "static", "-I", os.path.join(ROOT, "include")]

# lib -> (sources, headers, extra nvcc flags, link libs)
TARGETS = {
    "libpoly.so": (["poly.cu"], ["common.cuh", "dense.cuh", "finalize.cuh", "csr.cuh", "aux.cuh", "tv.cuh", "small.cuh", "ctproj.cuh", "p2p.cuh", "nvls.cuh", "dsell.cuh", "tiled.cuh"],
                   [], ["-ldl"]),
    "libpolysynth.so": (["synth.cu"], [], ["-fmad=false"], []),
}


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> list[str]:
    built = []
    for lib, (srcs, hdrs, flags, libs) in TARGETS.items():
        out = os.path.join(HERE, lib)
        deps = [os.path.join(CSRC, f) for f in srcs + hdrs] + [
            os.path.join(ROOT, "include", "poly.h"), os.path.join(ROOT, "include", "polysynth.h"),
            os.path.abspath(__file__)]
        if not force and not _stale(out, deps):
            continue
        cmd = [NVCC] + ARCH + COMMON + flags + [os.path.join(CSRC, s) for s in srcs] + \
            ["-o", out + ".tmp"] + libs
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
        os.replace(out + ".tmp", out)
        built.append(out)
    return built


if __name__ == "__main__":
    b = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print("built:", b if b else "(up to date)")
