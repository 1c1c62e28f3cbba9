"""Build libskg.so (sm_100a) in-tree with nvcc; no torch JIT cache involved."""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT = PKG / "libskg.so"
BUILD = PKG.parent / "build" / "skg"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
          f"-I{PKG.parent / 'include'}", "--expt-relaxed-constexpr"]
# The sampler's fp64 arithmetic must be IEEE-exact operation by operation (numpy
# parity): no FMA contraction in that translation unit.
PER_FILE = {
    "sampler.cu": ["--fmad=false"],
    "capi.cu": ["--fmad=false"],
    "gcn.cu": [],
    "gemm_tc.cu": [],
}


def nvcc() -> str:
    p = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(p).exists():
        raise RuntimeError("nvcc not found")
    return p


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("build failed: " + " ".join(cmd))
    return r.stdout + r.stderr


def sources():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))


def needs_build() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    deps = sources() + sorted(CSRC.glob("*.h")) + sorted(CSRC.glob("*.cuh")) + \
        sorted((PKG.parent / "include").glob("*.h"))
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> Path:
    if not force and not needs_build():
        return OUT
    BUILD.mkdir(parents=True, exist_ok=True)
    objs = []
    nv = nvcc()
    for src in sources():
        obj = BUILD / (src.name + ".o")
        if src.suffix == ".cu":
            cmd = [nv, *ARCH, *COMMON, *PER_FILE.get(src.name, []), "-Xptxas", "-v",
                   "-c", str(src), "-o", str(obj)]
        else:
            cmd = ["g++", "-O3", "-std=c++17", "-fPIC", f"-I{PKG.parent / 'include'}",
                   "-c", str(src), "-o", str(obj)]
        log = _run(cmd)
        if verbose:
            print(log)
        objs.append(str(obj))
    tmp = OUT.with_suffix(".so.tmp")
    _run([nv, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *objs])
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print(OUT)
