"""Build the native extension in-tree: csrc/*.cu -> librgbdseg_b200.so.

Plain nvcc (no torch JIT cache, so the .so travels with the repo snapshot):
  -gencode arch=compute_100a,code=sm_100a   B200 only
  -fmad=false --prec-div=true --prec-sqrt=true
        bit parity with the reference's numba FP64 (no FMA contraction,
        IEEE division/sqrt; SURVEY.md §7 "Hard parts" 1)
  -lineinfo                                 ncu source view
ptxas resource usage (-Xptxas -v) is kept in build/ptxas.log.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "librgbdseg_b200.so"
BUILD = ROOT / "build" / "native"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false", "--prec-div=true", "--prec-sqrt=true",
    "-Xcompiler", "-fPIC,-O2",
    "-Xptxas", "-v",
    "-I", str(ROOT / "include"),
]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; cannot build the sm_100a extension")


def sources():
    return sorted(CSRC.glob("*.cu"))


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "rgbdseg_b200.h",
                                                                 Path(__file__)]
    return any(p.stat().st_mtime > t for p in deps if p.exists())


def build(force: bool = False, verbose: bool = False, defines=(), out: Path | None = None) -> Path:
    """Compile csrc/*.cu into `out` (default: the in-tree librgbdseg_b200.so).
    `defines` (e.g. ["PBAS_MIN_BLOCKS=6"]) builds tuning variants."""
    if out is None and not defines and not force and not _stale():
        return LIB
    lib_out = Path(out) if out is not None else LIB
    build_dir = BUILD if not defines else BUILD / ("v_" + "_".join(d.replace("=", "") for d in defines))
    nvcc = _nvcc()
    build_dir.mkdir(parents=True, exist_ok=True)
    dflags = [f"-D{d}" for d in defines]

    def compile_one(src: Path):
        obj = build_dir / (src.stem + ".o")
        cmd = [nvcc, *NVCC_FLAGS, *dflags, "-c", str(src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr}")
        return obj, r.stderr

    jobs = min(len(sources()), os.cpu_count() or 4)
    with ThreadPoolExecutor(max_workers=jobs) as ex:
        results = list(ex.map(compile_one, sources()))
    (build_dir / "ptxas.log").write_text("".join(log for _, log in results))
    tmp = lib_out.with_suffix(".so.tmp")
    cmd = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(tmp)]
    cmd += [str(o) for o, _ in results]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, lib_out)
    if verbose:
        print(f"built {lib_out}", file=sys.stderr)
    return lib_out


def build_capi_demo(verbose: bool = False) -> Path:
    """examples/capi_demo: a plain C host of the C-ABI (no Python), linked
    against the in-tree library (rpath $ORIGIN/../paper_2002_00250_b200)."""
    src = ROOT / "examples" / "capi_demo.c"
    out = ROOT / "examples" / "capi_demo"
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        raise RuntimeError("no C compiler for examples/capi_demo.c")
    cmd = [cc, "-O2", "-std=c11", "-Wall", "-Wextra", "-o", str(out), str(src),
           "-L", str(PKG), "-lrgbdseg_b200", "-Wl,-rpath,$ORIGIN/../paper_2002_00250_b200"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"capi_demo build failed:\n{r.stderr}")
    if verbose:
        print(f"built {out}", file=sys.stderr)
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
