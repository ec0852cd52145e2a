"""Build libspmvtune_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2411_10143_b200.build [--force] [-v]

Each translation unit compiles to build/<name>.o (in parallel), then links
into paper_2411_10143_b200/libspmvtune_b200.so with a static CUDA runtime so
the library has no dependency on the toolkit's shared cudart at run time.
The SpMV unit is compiled with -fmad=false: its kernels reproduce the
reference's rounded-product-then-add order bit-for-bit.
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build"
LIB = PKG / "libspmvtune_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
          "-Xptxas", "-warn-spills", f"-I{ROOT / 'include'}"]
SOURCES = {
    "matrix.cu": [],
    "spmv.cu": ["-fmad=false"],
    "convert.cu": [],
    "features.cu": [],
    "krylov.cu": [],
    "generate.cu": [],
    "forest.cpp": [],
    "mmio.cu": [],
    "driver.cu": [],
    "peer.cu": [],
}


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _deps_newer(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + [ROOT / "include" / "spmvtune_b200.h", Path(__file__)]
    cc = nvcc()

    def compile_one(item):
        name, extra = item
        src = CSRC / name
        obj = BUILD / (src.stem + ".o")
        if not force and not _deps_newer(obj, [src] + headers):
            return obj
        cmd = [cc, *ARCH, *COMMON, *extra, "-c", str(src), "-o", str(obj)]
        if name.endswith(".cpp"):
            cmd = [cc, *ARCH, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", f"-I{ROOT / 'include'}",
                   "-c", str(src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), flush=True)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {name}:\n{res.stdout}\n{res.stderr}")
        if verbose and res.stderr.strip():
            print(res.stderr, flush=True)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, SOURCES.items()))
    if force or _deps_newer(LIB, objs):
        cmd = [cc, *ARCH, "-shared", "-cudart", "static", "-o", str(LIB), *map(str, objs)]
        if verbose:
            print(" ".join(cmd), flush=True)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    return LIB


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args(argv)
    print(build(force=a.force, verbose=a.verbose))


if __name__ == "__main__":
    sys.exit(main())
