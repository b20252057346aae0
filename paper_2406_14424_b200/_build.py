"""In-tree build of the sm_100a C-ABI library (libgearserve_b200.so).

nvcc cross-compiles for sm_100a without a GPU, so this runs in the CPU
container; the resulting .so travels to the GPU box with the repo snapshot.
Objects are rebuilt only when a source or header is newer.
"""

from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
BUILD = PKG / "_objs"
LIB = PKG / "libgearserve_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
              "--expt-relaxed-constexpr"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: cannot build libgearserve_b200.so")


def _sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _headers() -> list[Path]:
    return sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h"))


def build(verbose: bool = False, force: bool = False, phase_timing: bool = False,
          defines: tuple = (), tag: str = "") -> Path:
    """Compile every kernel source for sm_100a and link the shared library.
    phase_timing: a separate build (libgearserve_b200_phases.so, objects in
    _objs_phases/) whose kernels stamp %globaltimer at phase boundaries
    (GS_PHASE_TIMING; read back with gs_debug_phases) for tools/phase_probe.py."""
    nvcc = _nvcc()
    build_dir = BUILD.with_name("_objs_phases" + tag) if phase_timing else BUILD
    lib_path = LIB.with_name(f"libgearserve_b200_phases{tag}.so") if phase_timing else LIB
    extra = (["-DGS_PHASE_TIMING"] if phase_timing else []) + [f"-D{d}" for d in defines]
    if defines and not phase_timing:
        raise ValueError("experiment defines are for phase-timing builds only")
    build_dir.mkdir(exist_ok=True)
    hdr_mtime = max((p.stat().st_mtime for p in _headers()), default=0.0)
    objs = []
    for src in _sources():
        obj = build_dir / (src.stem + ".o")
        objs.append(obj)
        if (not force and obj.exists()
                and obj.stat().st_mtime >= max(src.stat().st_mtime, hdr_mtime)):
            continue
        cmd = [nvcc, *ARCH, *NVCC_FLAGS, *extra, "-I", str(INCLUDE), "-c", str(src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    newest = max(o.stat().st_mtime for o in objs)
    if force or not lib_path.exists() or lib_path.stat().st_mtime < newest:
        tmp = lib_path.with_suffix(".so.tmp")
        cmd = [nvcc, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs)]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        os.replace(tmp, lib_path)
    return lib_path


TORCH_OPS_SRC = CSRC / "gs_torch_ops.cpp"
TORCH_OPS_LIB = PKG / "libgearserve_b200_torch.so"


def build_torch_ops(verbose: bool = False, force: bool = False) -> Path:
    """The torch operator library (TORCH_LIBRARY gearserve_b200): a thin
    host-only C++ shim over libgearserve_b200.so, compiled with g++ against
    torch's headers and linked to the kernel library by an $ORIGIN rpath."""
    import torch
    from torch.utils import cpp_extension as ce

    lib = build(verbose=verbose, force=force)
    newest = max(TORCH_OPS_SRC.stat().st_mtime, lib.stat().st_mtime,
                 max(p.stat().st_mtime for p in INCLUDE.glob("*.h")))
    if not force and TORCH_OPS_LIB.exists() and TORCH_OPS_LIB.stat().st_mtime >= newest:
        return TORCH_OPS_LIB
    cuda_home = Path(_nvcc()).resolve().parent.parent
    abi = int(torch._C._GLIBCXX_USE_CXX11_ABI)
    cmd = [os.environ.get("CXX", "g++"), "-O2", "-std=c++17", "-fPIC", "-shared",
           f"-D_GLIBCXX_USE_CXX11_ABI={abi}", "-DTORCH_API_INCLUDE_EXTENSION_H",
           str(TORCH_OPS_SRC), "-I", str(INCLUDE), "-I", str(cuda_home / "include")]
    for inc in ce.include_paths():
        cmd += ["-I", inc]
    for d in ce.library_paths():
        cmd += ["-L", d, f"-Wl,-rpath,{d}"]
    cmd += ["-L", str(PKG), "-lgearserve_b200", "-Wl,-rpath,$ORIGIN",
            "-lc10", "-lc10_cuda", "-ltorch", "-ltorch_cpu", "-ltorch_cuda",
            "-o", str(TORCH_OPS_LIB.with_suffix(".so.tmp"))]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(TORCH_OPS_LIB.with_suffix(".so.tmp"), TORCH_OPS_LIB)
    return TORCH_OPS_LIB


if __name__ == "__main__":
    print(build(verbose=True))
    print(build_torch_ops(verbose=True))
