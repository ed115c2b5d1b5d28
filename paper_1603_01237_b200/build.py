"""Builds libqoc_b200.so (all CUDA kernels + the C-ABI host driver) for sm_100a, in-tree.

Each translation unit compiles to its own object in parallel (the kernel TUs are
independent: the host driver calls them through the launchers of csrc/kernels.h), then one
nvcc link produces the shared library.  Objects are cached by mtime under _lib/obj/.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT = PKG / "_lib" / "libqoc_b200.so"
OBJ = PKG / "_lib" / "obj"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
          "-Xptxas", "-warn-spills"]
INCLUDE = PKG.parent / "include"


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _headers() -> list[Path]:
    return list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [INCLUDE / "qoc_gpu.h"]


def _obj(src: Path) -> Path:
    return OBJ / (src.stem + ".o")


def _stale_obj(src: Path, hdr_mtime: float) -> bool:
    o = _obj(src)
    return not o.exists() or o.stat().st_mtime < max(src.stat().st_mtime, hdr_mtime)


def stale() -> bool:
    if not OUT.exists():
        return True
    # per object (a source edited while an earlier build was compiling it leaves an object
    # older than its source but a library newer than both)
    hdr = max(p.stat().st_mtime for p in _headers())
    if any(_stale_obj(s, hdr) for s in sources()):
        return True
    t = OUT.stat().st_mtime
    return any(_obj(s).stat().st_mtime > t for s in sources())


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not stale():
        return OUT
    OBJ.mkdir(parents=True, exist_ok=True)
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    hdr = max(p.stat().st_mtime for p in _headers())
    todo = [s for s in sources() if force or _stale_obj(s, hdr)]

    def compile_one(src: Path) -> None:
        tmp = _obj(src).with_suffix(".o.tmp")
        cmd = [nvcc, *ARCH, *CFLAGS, "-I", str(INCLUDE), "-c", "-o", str(tmp), str(src)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        tmp.replace(_obj(src))

    with ThreadPoolExecutor(max_workers=max(1, min(len(todo), os.cpu_count() or 1))) as ex:
        for f in [ex.submit(compile_one, s) for s in todo]:
            f.result()
    tmp = OUT.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH, "-shared", "-o", str(tmp), *[str(_obj(s)) for s in sources()]]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    tmp.replace(OUT)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
