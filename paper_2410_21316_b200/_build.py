"""In-tree build of libdos.so (nvcc for sm_100a + g++ for the host side).

The built library lives next to this file so gpurun snapshots carry it to the
GPU box; nothing is installed into site-packages.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
BUILD = PKG / "_objs"
LIB = PKG / "libdos.so"

CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA_HOME / "bin" / "nvcc")
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]

CXXFLAGS = [
    "-O3", "-fPIC", "-std=c++17", "-g",
    "-ffp-contract=off", "-fno-fast-math", "-fno-math-errno", "-fno-trapping-math",
    "-Wall", "-Wno-unused-function",
    f"-I{CUDA_HOME / 'include'}", f"-I{INCLUDE}",
]
ISA_FLAGS = {
    "avx512": ["-mavx512f", "-mavx512bw", "-mavx512vl", "-mavx512dq", "-mprfchw", "-mprefer-vector-width=512"],
    "avx2": ["-mavx2", "-mf16c"],
    "generic": [],
}
NVCCFLAGS = [
    *GENCODE, "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
    "-Xcompiler", "-fPIC", "-Xptxas", "-v",
    f"-I{INCLUDE}",
]


def _sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp")) + sorted(CSRC.glob("*.h")) + sorted(
        CSRC.glob("*.inc")) + sorted(INCLUDE.glob("*.h"))


def _run(cmd: list[str], log) -> None:
    log.write("+ " + " ".join(cmd) + "\n")
    proc = subprocess.run(cmd, capture_output=True, text=True)
    log.write(proc.stdout)
    log.write(proc.stderr)
    if proc.returncode != 0:
        raise RuntimeError(f"build step failed ({proc.returncode}): {' '.join(cmd)}\n{proc.stderr[-4000:]}")


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(s.stat().st_mtime > t for s in _sources())


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile libdos.so in-tree; returns its path."""
    if not force and not needs_build():
        return LIB
    if shutil.which(NVCC) is None and not Path(NVCC).exists():
        raise RuntimeError(f"nvcc not found at {NVCC}")
    BUILD.mkdir(exist_ok=True)
    logf = BUILD / "build.log"
    with open(logf, "w") as log:
        objs = []
        o = BUILD / "dos_cuda.o"
        _run([NVCC, *NVCCFLAGS, "-c", str(CSRC / "dos_cuda.cu"), "-o", str(o)], log)
        objs.append(o)
        for name in ("dos_host", "dos_exec", "dos_ipc"):
            o = BUILD / f"{name}.o"
            _run(["g++", *CXXFLAGS, "-c", str(CSRC / f"{name}.cpp"), "-o", str(o)], log)
            objs.append(o)
        for isa, flags in ISA_FLAGS.items():
            o = BUILD / f"dos_host_{isa}.o"
            _run(["g++", *CXXFLAGS, *flags, f"-DDOS_ISA_NS={isa}", "-fopt-info-vec-optimized",
                  "-c", str(CSRC / "dos_host_isa.cpp"), "-o", str(o)], log)
            objs.append(o)
        tmp = LIB.with_suffix(".so.tmp")
        _run([NVCC, *GENCODE, "-shared", "-o", str(tmp), *map(str, objs), "-lpthread", "-ldl", "-lrt"], log)
        os.replace(tmp, LIB)
    if verbose:
        sys.stdout.write(logf.read_text())
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
