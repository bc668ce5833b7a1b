"""In-tree build of the native library ``lib/libexsum_b200.so`` (sm_100a).

Compiles the CUDA sources with ``nvcc -gencode arch=compute_100a,code=sm_100a
-lineinfo -O3`` and the host C++ with g++, links one shared library with a
static CUDA runtime (so it does not depend on the toolkit's libcudart at run
time), and leaves it next to this file so it travels with the repo snapshot.
nvcc cross-compiles: no GPU is needed to build.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
BUILD = PKG / "_build"
LIB = PKG / "lib" / "libexsum_b200.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = "/usr/bin/g++"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SOURCES = ["sum_kernels.cu", "synth.cu", "context.cu", "nccl_sum.cu"]
CXX_SOURCES = ["host_accumulators.cpp", "io.cpp", "host_sum.cpp", "host_tools.cpp"]
HEADERS = [CSRC / "exsum_core.h", CSRC / "host_sum.h", CSRC / "exsum_nvtx.h", INCLUDE / "exsum_b200.h"]


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _run(cmd: list[str], verbose: bool) -> None:
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def build(verbose: bool = False, force: bool = False, defines: tuple[str, ...] = (),
          lib: Path = LIB, build_dir: Path = BUILD) -> Path:
    """Build the library; ``defines`` (-D...) and a separate lib/build_dir give
    tuning variants without touching the default artefact."""
    build_dir.mkdir(parents=True, exist_ok=True)
    lib.parent.mkdir(parents=True, exist_ok=True)
    dflags = [f"-D{d}" for d in defines if not d.startswith("NVCC:")]
    nvcc_extra = [d[5:] for d in defines if d.startswith("NVCC:")]
    objs: list[Path] = []
    common_inc = [f"-I{INCLUDE}", f"-I{CSRC}"]
    for src in CU_SOURCES:
        obj = build_dir / (src + ".o")
        objs.append(obj)
        if force or _stale(obj, [CSRC / src, *HEADERS]):
            _run([NVCC, *dflags, *nvcc_extra, *ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xptxas", "-v" if verbose else "-O3",
                  "-Xcompiler", "-fPIC,-ffp-contract=off,-fopenmp", *common_inc,
                  "-c", str(CSRC / src), "-o", str(obj)], verbose)
    for src in CXX_SOURCES:
        obj = build_dir / (src + ".o")
        objs.append(obj)
        if force or _stale(obj, [CSRC / src, *HEADERS]):
            _run([CXX, *dflags, "-std=c++17", "-O3" if src == "host_sum.cpp" else "-O2", "-fPIC",
                  "-pthread", "-Wall", "-Wextra", *common_inc, "-I/usr/local/cuda/include",
                  "-c", str(CSRC / src), "-o", str(obj)], verbose)
    if force or _stale(lib, objs):
        _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(lib), *map(str, objs),
              "-Xcompiler", "-fopenmp", "-lgomp", "-ldl", "-lpthread"], verbose)
    return lib


def build_variant(name: str, defines: tuple[str, ...], verbose: bool = False) -> Path:
    """Tuning variant: lib/variants/<name>.so (select with EXSUM_LIB=...)."""
    return build(verbose=verbose, defines=defines, lib=PKG / "lib" / "variants" / f"{name}.so",
                 build_dir=BUILD / "variants" / name)


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print(LIB)
