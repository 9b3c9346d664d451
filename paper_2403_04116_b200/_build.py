"""Build libxgauss.so (sm_100a) in-tree with nvcc.

The shared library is the product's only native artefact; it is built in
the package directory so it travels with the repository snapshot to the GPU
box.  ``xg_preprocess.cu`` and ``xg_project.cu`` are compiled with
``-fmad=false``: the per-Gaussian float64 projection (and the phantom
projector's ray samples) must round every product/sum as written so radii,
tile rects, depth keys and sample positions reproduce the oracle /
reference bit for bit; ``xg_tiles64.cu`` (the float64 plug-in kernels) too,
to round as the reference's Cython loop does.
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
LIB = PKG / "libxgauss.so"
OBJ = PKG / "csrc" / "_obj"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", f"-I{INCLUDE}"]
PER_FILE = {"xg_preprocess.cu": ["-fmad=false"], "xg_project.cu": ["-fmad=false"], "xg_tiles64.cu": ["-fmad=false"]}
SOURCES = ["xg_common.cu", "xg_preprocess.cu", "xg_sort.cu", "xg_bin.cu", "xg_composite.cu", "xg_optim.cu", "xg_ssim.cu", "xg_project.cu", "xg_tiles64.cu", "xg_dp.cu"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def _deps() -> list[Path]:
    return [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + [INCLUDE / "xgauss.h"]


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in _deps())


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return LIB
    OBJ.mkdir(parents=True, exist_ok=True)
    cc = nvcc()

    def compile_one(src: str) -> Path:
        out = OBJ / (Path(src).stem + ".o")
        cmd = [cc, *ARCH, *COMMON, *PER_FILE.get(src, []), "-c", str(CSRC / src), "-o", str(out)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        return out

    with ThreadPoolExecutor(max_workers=min(8, len(SOURCES))) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [cc, *ARCH, "-shared", "-o", str(tmp), *map(str, objs)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


def variant_path(name: str) -> Path:
    return PKG / "csrc" / "_variants" / f"libxgauss_{name}.so"


def build_variant(name: str, defines: list[str]) -> Path:
    """A tuning build of the library with extra -D flags (development aid:
    loaded instead of libxgauss.so when XG_LIB_VARIANT=name)."""
    out_dir = PKG / "csrc" / "_variants" / name
    out_dir.mkdir(parents=True, exist_ok=True)
    cc = nvcc()
    dflags = [f"-D{d}" for d in defines]

    def compile_one(src: str) -> Path:
        out = out_dir / (Path(src).stem + ".o")
        cmd = [cc, *ARCH, *COMMON, *dflags, *PER_FILE.get(src, []), "-c", str(CSRC / src), "-o", str(out)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        return out

    with ThreadPoolExecutor(max_workers=min(8, len(SOURCES))) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    lib = variant_path(name)
    r = subprocess.run([cc, *ARCH, "-shared", "-o", str(lib), *map(str, objs)], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{r.stdout}\n{r.stderr}")
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
