"""In-tree build of the native pieces (no JIT cache: the .so files travel to
the GPU box with the repo snapshot).

* ``libkvq.so``        -- the sm_100a kernels + C ABI (include/kvq.h)
* ``oracle/libkvq_oracle.so`` -- the CPU restatement used only by tests and the
  bench's CPU-baseline leg.
"""
from __future__ import annotations

import os
import subprocess
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
REPO = PKG_DIR.parent
CSRC = PKG_DIR / "csrc"
LIB_PATH = PKG_DIR / "libkvq.so"
ORACLE_DIR = REPO / "oracle"
ORACLE_LIB = ORACLE_DIR / "libkvq_oracle.so"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
]


def _nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def _stale(target: Path, sources) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(s).stat().st_mtime > t for s in sources)


def build_kernels(force: bool = False, verbose: bool = False) -> Path:
    sources = sorted(CSRC.glob("*.cu"))
    headers = sorted(CSRC.glob("*.cuh")) + [REPO / "include" / "kvq.h"]
    if force or _stale(LIB_PATH, sources + headers):
        cmd = [_nvcc(), *NVCC_FLAGS, "-I", str(REPO / "include"), "-o", str(LIB_PATH),
               *map(str, sources)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.run(cmd, check=True)
    return LIB_PATH


def source_hash() -> str:
    """Hash of everything that determines libkvq.so's code (CUDA sources, the
    ABI header, the nvcc flags): ties an ncu capture to the build it measured."""
    import hashlib
    h = hashlib.sha256(" ".join(NVCC_FLAGS).encode())
    for f in sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + [REPO / "include" / "kvq.h"]:
        h.update(f.name.encode())
        h.update(f.read_bytes())
    return h.hexdigest()[:16]


def build_oracle(force: bool = False) -> Path:
    src = [ORACLE_DIR / "kvq_oracle.c", ORACLE_DIR / "kvq_oracle.h"]
    if force or _stale(ORACLE_LIB, src):
        subprocess.run(["make", "-s", "-C", str(ORACLE_DIR), "-B" if force else "all"], check=True)
    return ORACLE_LIB


def build_all(force: bool = False) -> None:
    build_kernels(force=force)
    build_oracle(force=force)


if __name__ == "__main__":
    build_all(force=True)
