"""Build the native library in-tree: paper_1601_05052_b200/libdedisp_b200.so.

nvcc, sm_100a only (``-gencode arch=compute_100a,code=sm_100a``), ``-lineinfo``
for ncu source views, and deliberately WITHOUT --use_fast_math: the kernels
must keep IEEE round-to-nearest fp32 adds with denormals preserved
(-ftz=false is nvcc's default) to stay bit-identical to the reference.
The CUDA runtime is linked statically so the library loads without torch.

    python -m paper_1601_05052_b200.build        # or __graft_entry__.build()
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libdedisp_b200.so")
LIB_CHECKED = os.path.join(PKG, "libdedisp_b200_checked.so")
SOURCES = ["table.cu", "dedisp.cu", "abi.cu", "tuner.cu", "ingest.cu", "stream.cu", "host.cpp"]
HEADERS = ["common.cuh", "internal.hpp", "regwin_dispatch.cuh", "schedules.inc"]
PUBLIC = [os.path.join(ROOT, "include", "dedisp_b200.h"),
          os.path.join(ROOT, "include", "dedisp", "b200.hpp")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-Xptxas", "-v",
         "-I" + os.path.join(ROOT, "include"), "--expt-relaxed-constexpr"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def gen_dispatch() -> None:
    """Regenerate csrc/regwin_dispatch.cuh when its generator changed."""
    gen = os.path.join(CSRC, "gen_dispatch.py")
    out = os.path.join(CSRC, "regwin_dispatch.cuh")
    if _stale(out, [gen]):
        r = subprocess.run([sys.executable, gen], capture_output=True, text=True, check=True)
        with open(out, "w") as f:
            f.write(r.stdout)


def build(force: bool = False, verbose: bool = False, checked: bool = False,
          defines=(), out: str = None) -> str:
    """checked=True: libdedisp_b200_checked.so, the same library with every
    staged shared-memory read, bulk copy and output store bounds-checked on
    the device (-DDDB_CHECKED; dd_debug_violations) -- the memcheck stand-in
    (tests/test_gpu_checked.py).  defines/out: an A/B build of the same
    sources with extra -D macros into `out` (tools/ab_build.py)."""
    gen_dispatch()
    extra = (["-DDDB_CHECKED"] if checked else []) + ["-D" + d for d in defines]
    if out:
        tag = os.path.splitext(os.path.basename(out))[0]
        objdir = os.path.join(PKG, "build_ab", tag)
        lib = out
    else:
        objdir = os.path.join(PKG, "build_checked" if checked else "build")
        lib = LIB_CHECKED if checked else LIB
    os.makedirs(objdir, exist_ok=True)
    deps_common = [os.path.join(CSRC, h) for h in HEADERS] + PUBLIC + [__file__]
    objs = []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(objdir, src + ".o")
        objs.append(obj)
        if force or _stale(obj, [path] + deps_common):
            if src.endswith(".cu"):
                cmd = [nvcc()] + ARCH + FLAGS + extra + ["-c", path, "-o", obj]
            else:  # host-only C++ (the C++20 drop-in API and the tuner)
                cmd = [nvcc(), "-x", "c++", "-O3", "-std=c++20", "-Xcompiler", "-fPIC,-O3,-Wall",
                       "-I" + os.path.join(ROOT, "include"), "-c", path, "-o", obj]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {src}")
            if verbose:
                sys.stderr.write(r.stderr)
            with open(obj + ".ptxas.txt", "w") as f:
                f.write(r.stderr)
    if force or _stale(lib, objs):
        cmd = [nvcc()] + ARCH + ["-shared", "-o", lib] + objs + ["-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc link failed")
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv,
                checked="--checked" in sys.argv))
