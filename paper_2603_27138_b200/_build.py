"""Native build: compile the sm_100a kernels + C ABI into libscout_b200.so (in-tree).

nvcc cross-compiles for sm_100a without a GPU. Objects are rebuilt when their
source or a header is newer; the library lands next to this file so it travels
to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
ROOT = PKG.parent
OBJ = PKG / "_obj"
LIB = PKG / "libscout_b200.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX", "g++")
CUDA_INC = "/usr/local/cuda/include"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
           "-diag-suppress", "177", f"-I{ROOT / 'include'}"]


def _headers() -> list[Path]:
    return sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + sorted((ROOT / "include").glob("*.h"))


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build_native(force: bool = False, verbose: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    srcs = sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))
    hdrs = _headers()
    objs, cmds = [], []
    for src in srcs:
        obj = OBJ / (src.name + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + hdrs):
            cmd = [NVCC, *ARCH, *NVFLAGS, "-c", str(src), "-o", str(obj)]
            if src.suffix == ".cpp":  # host-only C++: the system compiler
                cmd = [CXX, "-O3", "-std=c++17", "-fPIC", "-Wall", "-pthread", f"-I{CUDA_INC}", f"-I{ROOT / 'include'}",
                       "-c", str(src), "-o", str(obj)]
            if verbose:
                print(" ".join(cmd))
            cmds.append(cmd)
    # one compiler process per stale source, all at once (the kernels are
    # independent translation units)
    procs = [subprocess.Popen(cmd) for cmd in cmds]
    failed = [" ".join(c) for c, p in zip(cmds, procs) if p.wait() != 0]
    if failed:
        raise subprocess.CalledProcessError(1, failed[0])
    if force or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-cudart", "static", "-Xcompiler", "-pthread"]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    return LIB


def build_oracle(verbose: bool = False) -> None:
    """Build the CPU checkers under oracle/ (test infrastructure, not the product)
    and, where the reference headers exist, the drop-in proof binaries
    tests/cpp/_bin/test_dropin_engine (the reference engine with the
    INTEGRATION.md §1 call swaps, linked to libscout_b200.so) and
    tests/cpp/_bin/test_tier_cache (the C++ TieredKvCache drop-in beside the
    reference's)."""
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle")], check=True,
                   stdout=None if verbose else subprocess.DEVNULL)
    subprocess.run(["make", "-s", "-C", str(ROOT / "tests" / "cpp")], check=True,
                   stdout=None if verbose else subprocess.DEVNULL)


if __name__ == "__main__":
    build_native(verbose=True)
    build_oracle(verbose=True)
