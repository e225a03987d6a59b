"""In-tree build of liblemo.so (sm_100a) with plain nvcc.

`python -m paper_2501_09767_b200.build` compiles every csrc/*.cu into one
shared library next to this file.  nvcc cross-compiles without a GPU, so
this runs in the CPU container as well as on the GPU box.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
# LEMO_BUILD_TAG builds an A/B variant (own object dir, liblemo_<tag>.so) of the same sources
_TAG = os.environ.get("LEMO_BUILD_TAG", "")
LIB = PKG / (f"liblemo_{_TAG}.so" if _TAG else "liblemo.so")
OBJ = PKG / (f"_build_{_TAG}" if _TAG else "_build")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills"] + os.environ.get("LEMO_EXTRA_NVCC_FLAGS", "").split()


def _nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _stale(src: Path, obj: Path) -> bool:
    if not obj.exists():
        return True
    deps = [src, *CSRC.glob("*.cuh"), *CSRC.glob("*.h"), PKG.parent / "include" / "lemo.h"]
    t = obj.stat().st_mtime
    return any(d.exists() and d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    nvcc = _nvcc()
    stamp = OBJ / "flags.txt"  # a flag change (e.g. LEMO_EXTRA_NVCC_FLAGS) rebuilds everything
    if not stamp.exists() or stamp.read_text() != " ".join(FLAGS):
        force = True
        stamp.write_text(" ".join(FLAGS))
    inc = ["-I", str(CSRC), "-I", str(PKG.parent / "include")]
    jobs = []
    for src in sources():
        obj = OBJ / (src.stem + ".o")
        if force or _stale(src, obj):
            jobs.append([nvcc, *ARCH, *FLAGS, *inc, "-c", str(src), "-o", str(obj)])

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and r.stderr.strip():
            print(r.stderr, file=sys.stderr)
        return r

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        list(ex.map(run, jobs))
    objs = [str(OBJ / (s.stem + ".o")) for s in sources()]
    if jobs or force or not LIB.exists():
        run([nvcc, *ARCH, "-shared", "-o", str(LIB), *objs])
    return LIB


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print(LIB)
