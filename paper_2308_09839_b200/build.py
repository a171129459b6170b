"""Build libfem.so (CUDA sm_100a, FP64) in-tree with nvcc.

    python -m paper_2308_09839_b200.build [--force]

The shared library is the C ABI of include/fem.h.  NCCL (headers + libnccl.so.2) comes from the
nvidia-nccl wheel bundled with torch; it is linked with an rpath so no LD_LIBRARY_PATH is needed.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libfem.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir() -> str:
    cands = []
    for sp in {sysconfig.get_paths()["purelib"], sysconfig.get_paths()["platlib"]}:
        cands.append(os.path.join(sp, "nvidia", "nccl"))
    try:
        import nvidia.nccl  # type: ignore
        cands.insert(0, os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else
                     list(nvidia.nccl.__path__)[0])
    except Exception:
        pass
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return c
    raise RuntimeError("nccl.h not found (expected the nvidia-nccl wheel next to torch)")


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "fem.h")])


def _needs_build(force: bool) -> bool:
    if force or not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in _sources() + _headers() + [__file__])


def build(force: bool = False, verbose: bool = False) -> str:
    if not _needs_build(force):
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    nd = nccl_dir()
    common = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(nd, "include"),
                     "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]
    if verbose:
        common += ["-Xptxas", "-v"]
    common += os.environ.get("FEM_NVCC_FLAGS", "").split()  # experiments only (e.g. -DFEM_EL_TY=12)
    objs = []

    def compile_one(src):
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        cmd = [NVCC] + common + ["-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        return obj, r.stderr

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        for obj, log in ex.map(compile_one, _sources()):
            objs.append(obj)
            if verbose and log:
                sys.stderr.write(log)
    libdir = os.path.join(nd, "lib")
    link = [NVCC] + ARCH + ["-shared", "-o", LIB + ".tmp"] + objs + [
        "-L" + libdir, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + libdir, "-lcudart_static",
        "-ldl", "-lrt", "-lpthread"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
