"""Build the sm_100a shared library `_lib/liblsopc_b200.so` in-tree.

    python -m paper_2303_12529_b200.build          # incremental
    python -m paper_2303_12529_b200.build --force

nvcc cross-compiles for sm_100a without a GPU.  Objects are rebuilt when the
source or any csrc header is newer.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
# LSB_OUT / LSB_DEFINES build experiment variants into another directory
# (e.g. LSB_OUT=/tmp/v1 LSB_DEFINES="-DLSB_EXP_NOSTORE"); the package loads
# the default library unless LSOPC_B200_LIB points elsewhere.
OUT_DIR = Path(os.environ.get("LSB_OUT") or (PKG / "_lib"))
LIB = OUT_DIR / "liblsopc_b200.so"
EXTRA = os.environ.get("LSB_DEFINES", "").split()
INCLUDE = PKG.parent / "include"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
         "--expt-relaxed-constexpr", "-I", str(INCLUDE)]


def _sources():
    return sorted(CSRC.glob("*.cu"))


def _headers_mtime():
    hs = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list(INCLUDE.glob("*.h"))
    return max((h.stat().st_mtime for h in hs), default=0.0)


def build(force: bool = False, verbose: bool = False) -> Path:
    OUT_DIR.mkdir(parents=True, exist_ok=True)
    hdr = _headers_mtime()
    objs, jobs = [], []
    for src in _sources():
        obj = OUT_DIR / (src.stem + ".o")
        objs.append(obj)
        if force or not obj.exists() or obj.stat().st_mtime < max(src.stat().st_mtime, hdr):
            jobs.append((src, obj))

    def compile_one(job):
        src, obj = job
        cmd = [NVCC, *ARCH, *FLAGS, *EXTRA, "-c", str(src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr}")
        return src.name, r.stderr

    if jobs:
        with ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            for name, err in ex.map(compile_one, jobs):
                if verbose and err:
                    print(f"== {name}\n{err}", file=sys.stderr)
    if jobs or not LIB.exists():
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-cudart", "static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
