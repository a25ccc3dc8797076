"""Build the sm_100a shared library in-tree (it travels to the GPU box).

    python -m paper_2604_19892_b200.build_native

One nvcc invocation: csrc/maspncg.cu (unity build) -> libmaspncg.so with the
CUDA runtime static.  -lineinfo keeps ncu's source view mapped to our code.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libmaspncg.so"
CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _sources():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "maspncg.h"]


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(s.stat().st_mtime > t for s in _sources())


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return LIB
    nvcc = CUDA_HOME / "bin" / "nvcc"
    cmd = [
        str(nvcc), *ARCH, "-O3", "-std=c++17", "-lineinfo", "-shared", "-Xcompiler", "-fPIC",
        "-Xptxas", "-v" if verbose else "-O3",
        "-I", str(PKG.parent / "include"),
        "-o", str(LIB) + ".tmp", str(CSRC / "maspncg.cu"),
        "-L", str(CUDA_HOME / "lib64"),
        "-Xlinker", f"-rpath,{CUDA_HOME / 'lib64'}",
    ]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libmaspncg.so")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(str(LIB) + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)


FP64_PEAK = PKG.parent / "tools" / "micro" / "fp64_peak"


def build_fp64_peak() -> Path:
    """The FP64 FMA peak probe bench.py runs for the FP64 rooflines
    (tools/micro/fp64_peak.cu; a diagnostic binary, not part of the library)."""
    src = FP64_PEAK.with_suffix(".cu")
    if FP64_PEAK.exists() and FP64_PEAK.stat().st_mtime >= src.stat().st_mtime:
        return FP64_PEAK
    cmd = [str(CUDA_HOME / "bin" / "nvcc"), *ARCH, "-O3", "-o", str(FP64_PEAK), str(src)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed for fp64_peak:\n" + res.stderr[-2000:])
    return FP64_PEAK
