"""Build libdk.so (the C-ABI library) in-tree with nvcc for sm_100a.

Usage:  python -m paper_1510_02148_b200.csrc.build   (or build() from __graft_entry__)
The .so lands next to this file's package (paper_1510_02148_b200/_lib/libdk.so) so it
travels with the repository snapshot to the GPU box.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

CSRC = Path(__file__).resolve().parent
PKG = CSRC.parent
ROOT = PKG.parent
OUT_DIR = PKG / "_lib"
LIB = OUT_DIR / "libdk.so"

SOURCES = ["dk_device.cu", "dk_kernels.cu", "dk_coarse.cu", "dk_dense.cu", "dk_profile.cu", "dk_setup.cu", "dk_api.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the B200 library cannot be built")


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) \
        + [ROOT / "include" / "dk.h"]
    return any(p.stat().st_mtime > t for p in deps if p.exists())


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    OUT_DIR.mkdir(parents=True, exist_ok=True)
    objs = []
    tmp = OUT_DIR / "obj"
    tmp.mkdir(exist_ok=True)
    cc = nvcc()
    cmds = []
    for src in SOURCES:
        obj = tmp / (Path(src).stem + ".o")
        cmd = [cc, "-c", str(CSRC / src), "-o", str(obj), "-O3", "-std=c++17",
               "-Xcompiler", "-fPIC", "-I", str(ROOT / "include")]
        if src.endswith(".cu"):
            cmd += ARCH + ["-lineinfo", "-Xptxas", "-O3,-v" if verbose else "-O3"]
        else:
            cmd = [shutil.which("g++") or "g++", "-c", str(CSRC / src), "-o", str(obj), "-O3",
                   "-std=c++17", "-fPIC", "-I", str(ROOT / "include")]
        cmds.append(cmd)
        objs.append(str(obj))

    def compile_one(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
        if verbose or r.returncode:
            print(r.stdout, flush=True)
        r.check_returncode()

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 1)) as ex:
        list(ex.map(compile_one, cmds))
    tmp_lib = LIB.with_suffix(".so.tmp")
    cmd = [cc, "-shared", *ARCH, "-o", str(tmp_lib), *objs, "-cudart", "static"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(tmp_lib, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
