"""In-tree build of libmfreg_cuda.so for sm_100a (nvcc direct; no JIT cache).

Every translation unit is compiled with ``--fmad=false`` so the device
arithmetic keeps the reference's separately rounded multiply/add order
(DESIGN.md §3); kernels that may contract call fma() explicitly.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libmfreg_cuda.so")
SOURCES = ["kernels.cu", "fused.cu", "hv_fast.cu", "hv3.cu", "ev_fast.cu", "cg.cu", "objective.cu", "solvers.cu", "io.cu", "capi.cu", "api.cu", "slab.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
                     "-Xptxas", "-O3", "--expt-relaxed-constexpr"]


def _nvcc() -> str:
    for c in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.exists(c) or c == "nvcc":
            return c
    return "nvcc"


def _stale(obj: str, deps: list[str]) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def variant_lib(variant: str) -> str:
    """Path of an experiment build (scripts/variants.py): libmfreg_cuda_<variant>.so."""
    return os.path.join(HERE, "variants", f"libmfreg_cuda_{variant}.so")  # travels to the GPU box


def build(verbose: bool = False, force: bool = False, variant: str = "", defines: tuple = ()) -> str:
    """Compile the library; `variant`/`defines`: an A/B experiment build with extra -D flags
    (loaded by the package when MFREG_LIB_VARIANT=<variant>)."""
    obj_dir = os.path.join(OBJ, variant) if variant else OBJ
    lib_path = variant_lib(variant) if variant else LIB
    flags = NVCC_FLAGS + [f"-D{d}" for d in defines]
    os.makedirs(obj_dir, exist_ok=True)
    os.makedirs(os.path.dirname(lib_path), exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(HERE, "..", "include", "mfreg_cuda.h"))
    jobs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        if not os.path.exists(s):
            continue
        o = os.path.join(obj_dir, src.replace(".cu", ".o"))
        if force or variant or _stale(o, [s, *headers, __file__]):
            jobs.append([_nvcc(), *flags, "-c", s, "-o", o])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stdout or r.stderr):
            print(r.stdout, r.stderr)

    with cf.ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
        list(ex.map(run, jobs))
    objs = [os.path.join(obj_dir, s.replace(".cu", ".o")) for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    if jobs or not os.path.exists(lib_path) or _stale(lib_path, objs):
        run([_nvcc(), *ARCH, "-shared", "-o", lib_path, *objs, "-lcudart"])
    return lib_path


if __name__ == "__main__":
    print(build(verbose=True))
