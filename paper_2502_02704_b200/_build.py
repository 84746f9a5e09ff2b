"""In-tree build of libpbgk.so (sm_100a) with nvcc.

The shared library is the product: every hot kernel and the C ABI of
include/pbgk.h.  It is built in place (paper_2502_02704_b200/lib/) so the
snapshot that travels to the GPU box carries it.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "lib"
LIB = LIBDIR / "libpbgk.so"
SOURCES = ["sweep.cu", "sweep_a.cu", "sweep_b.cu", "sweep_c.cu", "finalize.cu", "fluid.cu", "fsweep.cu", "msweep.cu", "esweep.cu", "marginal.cu", "capi.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         "-I", str(ROOT / "include")]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = list(CSRC.glob("*")) + [ROOT / "include" / "pbgk.h"]
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False, csrc: Path | None = None,
          out: Path | None = None) -> Path:
    """Compile the CUDA sources to lib/libpbgk.so (skipped when up to date).

    ``csrc`` / ``out`` let development builds compile another source tree
    (e.g. the previous revision, for A/B timing) to another file."""
    global CSRC, LIB
    if csrc is not None:
        CSRC, LIB = Path(csrc), Path(out)
        force = True
    if not force and not _stale():
        return LIB
    LIBDIR.mkdir(exist_ok=True)
    cc = nvcc()
    objs = []

    def one(src):
        obj = LIB.parent / (LIB.stem + "_" + Path(src).stem + ".o")
        defs = os.environ.get("PBGK_NVCC_DEFS", "").split()  # dev A/B variants
        cmd = [cc, *ARCH, *FLAGS, *defs, "-Xptxas", "-v", "-c", str(CSRC / src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed for %s:\n%s" % (src, r.stderr))
        (LIB.parent / (LIB.stem + "_" + Path(src).stem + ".ptxas.txt")).write_text(r.stderr)
        return obj

    srcs = [f for f in SOURCES if (CSRC / f).exists()]  # older trees (A/B builds) have fewer
    with cf.ThreadPoolExecutor(len(srcs)) as ex:
        objs = list(ex.map(one, srcs))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [cc, *ARCH, "-shared", "-o", str(tmp), *map(str, objs)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n" + r.stderr)
    os.replace(tmp, LIB)
    for o in objs:  # every build recompiles all sources; keep the snapshot lean
        Path(o).unlink(missing_ok=True)
    if verbose:
        print("built", LIB)
    return LIB


if __name__ == "__main__":
    import sys
    if len(sys.argv) == 3:  # python _build.py <csrc dir> <out .so>
        build(csrc=Path(sys.argv[1]), out=Path(sys.argv[2]), verbose=True)
    else:
        build(force=True, verbose=True)
