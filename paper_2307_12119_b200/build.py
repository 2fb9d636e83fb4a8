"""In-tree build of the sm_100a library ``libgreentherm_b200.so``.

Every CUDA source is compiled with ``-gencode arch=compute_100a,code=sm_100a
-lineinfo`` by nvcc; host C++ sources go through nvcc's host compiler so the
static CUDA runtime is linked once. The shared object lands next to this file
(``paper_2307_12119_b200/libgreentherm_b200.so``) so it travels to the GPU box
with the repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
BUILD = PKG.parent / "build" / "obj"
LIB = PKG / "libgreentherm_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
            "-Xptxas", "-warn-spills"]
CXX_FLAGS = ["-O2", "-std=c++17", "-Xcompiler", "-fPIC,-Wall"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the B200 library cannot be built")


def _host_compiler() -> list[str]:
    # Link the system libstdc++ dynamically (a static copy inside the .so
    # clashes with the one Python/torch already loaded).
    for cand in ("/usr/bin/g++", shutil.which("g++")):
        if cand and Path(cand).exists():
            return ["-ccbin", cand]
    return []


def _sources() -> list[Path]:
    return sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cpp")))


def _headers() -> list[Path]:
    return sorted(list(CSRC.glob("*.h")) + list(CSRC.glob("*.hpp")) + list(CSRC.glob("*.cuh"))
                  + list(INCLUDE.glob("*.h")))


def _compile(src: Path, nvcc: str, hdr_mtime: float, objdir: Path = BUILD, extra: tuple = ()) -> Path:
    obj = objdir / (src.name + ".o")
    if obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, hdr_mtime):
        return obj
    # variant defines (-D...) reach the host sources too
    flags = (ARCH + CU_FLAGS + list(extra)) if src.suffix == ".cu" else CXX_FLAGS + [e for e in extra if e.startswith("-D")]
    cmd = [nvcc, *_host_compiler(), *flags, "-I", str(CSRC), "-I", str(INCLUDE), "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    return obj


def build(verbose: bool = False, variant: str | None = None, extra: tuple = ()) -> Path:
    """Build the library; ``variant`` + ``extra`` nvcc defines build a tuning
    variant to ``variants/libgreentherm_b200_<variant>.so`` (selected at run
    time with GT_B200_LIB) without touching the product library."""
    nvcc = _nvcc()
    objdir = BUILD if variant is None else BUILD.parent / f"obj_{variant}"
    lib = LIB if variant is None else PKG / f"libgreentherm_b200_v{variant}.so"
    objdir.mkdir(parents=True, exist_ok=True)
    lib.parent.mkdir(parents=True, exist_ok=True)
    hdr_mtime = max(p.stat().st_mtime for p in _headers())
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, nvcc, hdr_mtime, objdir, extra), srcs))
    newest = max(o.stat().st_mtime for o in objs)
    if lib.exists() and lib.stat().st_mtime >= newest:
        return lib
    LIB_ = lib
    tmp = LIB_.with_suffix(".so.tmp")
    cmd = [nvcc, *_host_compiler(), *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lpthread"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, LIB_)
    if verbose:
        print(f"built {LIB_}")
    return LIB_


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--variant":
        build(verbose=True, variant=sys.argv[2], extra=tuple(sys.argv[3:]))
    else:
        build(verbose=True)
    sys.exit(0)
