"""Build the in-tree native library ``libporeflow_b200.so`` (sm_100a).

Plain ``nvcc`` (no torch JIT cache): the ``.so`` lands next to this file so it
travels with the repository snapshot to the GPU box.  cuFFT is linked
dynamically by SONAME (``libcufft.so.11``) so the process shares the copy
PyTorch already loaded; the CUDA runtime is linked statically.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
ROOT = PKG.parent
LIB = PKG / "libporeflow_b200.so"
SOURCES = ["pf_plan.cu", "pf_stokes.cu", "pf_transport.cu", "pf_effective.cu", "pf_kernels.cu", "pf_fused.cu",
           "pf_fused_transport.cu", "pf_slab.cu", "pf_ops.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


# The kernel plugin and the cuFFT pipeline evaluate the reference's formulas in
# its order without FMA contraction (bit-exact pointwise kernels); the fused
# pipeline's transforms differ from pocketfft anyway, so it lets nvcc contract.
FMAD = {"pf_fused.cu": "true", "pf_fused_transport.cu": "true"}


def _flags(src: str = ""):
    return ARCH + ["-O3", "-lineinfo", f"--fmad={FMAD.get(src, 'false')}", "-std=c++17", "-Xcompiler",
                   "-fPIC,-O3", "-I", str(ROOT / "include"), "-Xptxas", "-v"] + (["-DNDEBUG"])


def sources():
    return [CSRC / s for s in SOURCES if (CSRC / s).exists()]


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = (list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h"))
            + [Path(__file__)])
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False, out: Path | None = None, defines=()) -> Path:
    """Compile every source and link the C-ABI library.  ``out``/``defines`` build a
    tuning variant (extra -D flags) next to the product library, for A/B timing via
    POREFLOW_B200_LIB; the product build uses neither."""
    lib = Path(out) if out else LIB
    if out is None and not force and not needs_build():
        return LIB
    cc = nvcc()
    objdir = PKG / "build" if out is None else PKG / "build" / ("v_" + lib.stem)
    objdir.mkdir(parents=True, exist_ok=True)
    extra = [f"-D{d}" for d in defines]

    def compile_one(src: Path):
        obj = objdir / (src.stem + ".o")
        cmd = [cc, "-c", str(src), "-o", str(obj)] + _flags(src.name) + extra
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr}")
        (objdir / (src.stem + ".ptxas.txt")).write_text(r.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, sources()))
    tmp = lib.with_suffix(".so.tmp")
    cmd = [cc, "-shared", "-o", str(tmp)] + [str(o) for o in objs] + ARCH + [
        "-L/usr/local/cuda/lib64", "-lcufft", "-Xlinker", "-rpath,/usr/local/cuda/lib64",
    ]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{r.stderr}")
    os.replace(tmp, lib)
    if verbose:
        print(f"built {lib} ({lib.stat().st_size / 1e6:.1f} MB)", file=sys.stderr)
    return lib


if __name__ == "__main__":
    # python _build.py [--force] [--variant NAME -DX=1 -DY=2 ...]
    args = sys.argv[1:]
    if "--variant" in args:
        name = args[args.index("--variant") + 1]
        defs = [a[2:] for a in args if a.startswith("-D")]
        build(verbose=True, out=PKG / "build" / f"lib_{name}.so", defines=defs)
    else:
        build(force="--force" in args, verbose=True)
