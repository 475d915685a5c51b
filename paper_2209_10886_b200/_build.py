"""Build libhsb200.so (sm_100a) in-tree with nvcc.

    python -m paper_2209_10886_b200._build [--force] [-v]

Objects are compiled in parallel into build/ and linked into
paper_2209_10886_b200/_lib/libhsb200.so (git-ignored, travels to the GPU box
with the gpurun snapshot).  NCCL comes from the nvidia-nccl wheel torch uses.
"""

from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(OUT_DIR, "libhsb200.so")
BUILD = os.path.join(ROOT, "build", "hsb200")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_paths():
    try:
        import nvidia.nccl as m  # the wheel torch links against
        base = list(m.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    except Exception:
        pass
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + glob.glob(os.path.join(ROOT, "include", "*.h")))


def _needs(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, debug: bool = False) -> str:
    """debug = True: libhsb200_debug.so, the device-checks build (-DHS_DEVICE_CHECKS:
    bounds asserts + spin watchdogs, hs_debug_check; HS_LIB=debug loads it)."""
    os.makedirs(OUT_DIR, exist_ok=True)
    build_dir = BUILD + ("_debug" if debug else "")
    lib_out = LIB.replace("libhsb200.so", "libhsb200_debug.so") if debug else LIB
    os.makedirs(build_dir, exist_ok=True)
    inc, lib = nccl_paths()
    common = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I", inc, "-I", os.path.join(ROOT, "include"),
              "--expt-relaxed-constexpr"] + (["-DHS_DEVICE_CHECKS"] if debug else [])
    hdrs = headers()
    jobs = []
    objs = []
    for src in sources():
        obj = os.path.join(build_dir, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _needs(obj, [src] + hdrs):
            cmd = [NVCC] + ARCH + common + ["-Xptxas", "-v" if verbose else "-O3", "-c", src, "-o", obj]
            if src.endswith(".cpp"):
                cmd = [NVCC] + ARCH + common + ["-x", "c++", "-c", src, "-o", obj]
            jobs.append(cmd)

    def run(cmd):
        p = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, p

    with cf.ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        for cmd, p in ex.map(run, jobs):
            if verbose or p.returncode:
                sys.stderr.write(" ".join(cmd) + "\n" + p.stdout + p.stderr)
            if p.returncode:
                raise RuntimeError(f"nvcc failed for {cmd[-3]}")
    if force or jobs or _needs(lib_out, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", lib_out] + objs + [
            "-L", lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + lib]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode:
            sys.stderr.write(" ".join(cmd) + "\n" + p.stdout + p.stderr)
            raise RuntimeError("link failed")
    return lib_out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, debug="--debug" in sys.argv))
