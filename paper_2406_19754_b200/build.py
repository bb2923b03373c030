"""Build libpsc.so in-tree: nvcc for sm_100a (B200), NCCL from the torch-bundled wheel.

    python paper_2406_19754_b200/build.py [--force]     (or __graft_entry__.build())
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libpsc.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_paths():
    """Headers + library of the NCCL that torch loads (one libnccl.so.2 per process)."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        inc, lib = os.path.join(base, "nccl", "include"), os.path.join(base, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
            return inc, lib
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def flags():
    inc, _ = nccl_paths()
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3,-ffp-contract=off", "-Xptxas", "-v",
                   "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc]


def _compile(src, defines=()):
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    deps = [src] + glob.glob(os.path.join(CSRC, "*.h")) + [os.path.join(ROOT, "include", "psc.h")]
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps):
        return obj, ""
    r = subprocess.run([NVCC] + flags() + list(defines) + ["-c", src, "-o", obj], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """Build libpsc.so (or, for experiments, `out` with extra -D defines in a separate object dir)."""
    global BUILD
    lib = out or LIB
    build_dir = BUILD if not out else os.path.join(HERE, "_build_" + os.path.basename(out).replace(".so", ""))
    saved = BUILD
    BUILD = build_dir
    try:
        return _build(force, verbose, lib, list(defines))
    finally:
        BUILD = saved


def _build(force, verbose, LIB, defines):
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    if force:
        for o in glob.glob(os.path.join(BUILD, "*.o")):
            os.remove(o)
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        res = list(ex.map(lambda f: _compile(f, defines), srcs))
    objs = [o for o, _ in res]
    if verbose:
        for _, log in res:
            if log:
                sys.stderr.write(log)
    if (not force and os.path.exists(LIB)
            and os.path.getmtime(LIB) >= max(os.path.getmtime(o) for o in objs)):
        return LIB
    _, nlib = nccl_paths()
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + [
        "-L", nlib, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{nlib}", "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


def build_checked(force: bool = False) -> str:
    """libpsc_checked.so: the same sources with device-side bounds checks (-DPSC_CHECKS),
    for test runs with PSC_LIB pointing at it (compute-sanitizer is not available on the
    GPU pool)."""
    return build(force=force, out=os.path.join(HERE, "libpsc_checked.so"), defines=["-DPSC_CHECKS"])


if __name__ == "__main__":
    if "--checked" in sys.argv:
        print(build_checked(force="--force" in sys.argv))
    else:
        print(build(force="--force" in sys.argv, verbose=True))
