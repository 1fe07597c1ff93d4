"""Build the sm_100a C-ABI library in-tree: ``_lib/libpipesched_b200.so``.

Plain nvcc, one translation unit per evaluator lane width compiled in parallel,
static CUDA runtime, ``-lineinfo`` for ncu source views.  Rebuilds only when a
source or header is newer than the library.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
LIBDIR = PKG / "_lib"
LIB = LIBDIR / "libpipesched_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr"]

SOURCES = ["ps_abi.cu", "ps_bound.cu", "ps_literal.cu"] + [f"ps_eval_{t}_m{m}.cu" for t in ("i32", "i64") for m in (0, 1)]


def _inputs():
    yield from CSRC.glob("*.cu")
    yield from CSRC.glob("*.cuh")
    yield from CSRC.glob("*.h")
    yield from INCLUDE.glob("*.h")
    yield Path(__file__)


def needs_build() -> bool:
    if not LIB.exists():
        return True
    built = LIB.stat().st_mtime
    return any(p.stat().st_mtime > built for p in _inputs())


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"command failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r


def build(force: bool = False, verbose: bool = False, defines=(), out: Path | None = None) -> Path:
    """Build the library; `defines`/`out` produce an experiment variant (tools/kexp.py) elsewhere."""
    lib = Path(out) if out else LIB
    if not force and not defines and lib == LIB and not needs_build():
        return LIB
    objdir = lib.parent / ("obj" if lib == LIB else "obj_" + lib.stem)
    objdir.mkdir(parents=True, exist_ok=True)

    def compile_one(src):
        obj = objdir / (Path(src).stem + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-I", str(INCLUDE), "-c", str(CSRC / src),
               "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        r = _run(cmd)
        if verbose:
            sys.stderr.write(r.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = lib.with_suffix(".so.tmp")
    _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs), "-ldl"])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs,
                out=Path(outs[0]) if outs else None))
