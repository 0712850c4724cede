"""Builds libfbf.so (the fbf C ABI: host C++ + sm_100a CUDA) in-tree.

    python -m paper_1811_02168_b200.build [--force] [--jobs N]

nvcc cross-compiles for sm_100a without a GPU. The 32 radius
specialisations of the fused kernel are split across several translation units
so they compile in parallel. The shared library is written next to this file
(git-ignored; it travels to the GPU box with the repo snapshot).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(ROOT, "build", "fbf")
LIB = os.path.join(HERE, "libfbf.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC,-O3", "-Xptxas", "-v",
                     f"-I{os.path.join(ROOT, 'include')}"]
CXX_FLAGS = ["-O3", "-std=c++20", "-fPIC", "-pthread", f"-I{os.path.join(ROOT, 'include')}"]
# host library + auxiliary kernels (period scan, brute filter, 8-bit I/O)
HOST_CU = ["fbf_api.cu", "fbf_scan.cu", "fbf_brute.cu"]
# radius ranges per kernel translation unit (big radii are the slow ones)
RADIUS_SPLITS = [(1, 8), (9, 12), (13, 15), (16, 18), (19, 21), (22, 24), (25, 26), (27, 28),
                 (29, 30), (31, 32)]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _deps() -> list[str]:
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "fbf.h")]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str], log: str) -> None:
    p = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + p.stdout + p.stderr)
    if p.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{p.stdout}{p.stderr}")


def _check_inlined(tasks) -> None:
    """The fused kernel's role lambdas must inline into the kernel: when code growth
    pushes one out of line, ptxas compiles it as a separate ABI function (its own
    'Function properties for _ZZN7fbf_dev16fbf_fused_kernel...' entry) with spilled
    loop state, and the kernel runs ~2x slower (seen on c1: 0.57 -> 0.31 of peak)."""
    bad = []
    for _, log in tasks:
        with open(log) as f:
            for line in f:
                if "Function properties for _ZZN7fbf_dev16fbf_fused_kernel" in line:
                    bad.append(line.split("for ", 1)[1].strip())
    if bad:
        raise RuntimeError("fused kernel role code compiled out of line (not inlined): " + ", ".join(bad[:4]))


def build(force: bool = False, jobs: int | None = None, verbose: bool = False, out: str | None = None,
          defines: list[str] | None = None, radius: int | None = None) -> str:
    """Builds libfbf.so. Dev options: `out` (another library path), `defines`
    (extra -D macros, e.g. FBF_SKIP_GEN), `radius` (specialise one radius only)."""
    lib = out or LIB
    deps = _deps()
    if not force and not _stale(lib, deps):
        return lib
    extra = [f"-D{d}" for d in (defines or [])]
    splits = RADIUS_SPLITS
    build_dir = BUILD
    if radius is not None:
        splits = [(radius, radius)]
        extra.append(f"-DFBF_DEV_RADIUS={radius}")
    if out or defines or radius is not None:
        build_dir = os.path.join(ROOT, "build", "fbf_dev_" + os.path.basename(lib).replace(".so", ""))
    os.makedirs(build_dir, exist_ok=True)
    nvcc = _nvcc()
    jobs = jobs or min(len(splits) + 3, os.cpu_count() or 4)
    tasks = []
    objs = []
    for lo, hi in splits:
        obj = os.path.join(build_dir, f"fbf_kernel_r{lo:02d}_{hi:02d}.o")
        objs.append(obj)
        tasks.append(([nvcc, *NVCC_FLAGS, *extra, f"-DFBF_R_LO={lo}", f"-DFBF_R_HI={hi}", "-c",
                       os.path.join(CSRC, "fbf_kernel_inst.cu"), "-o", obj], obj + ".log"))
    for src in HOST_CU:
        obj = os.path.join(build_dir, src.replace(".cu", ".o"))
        objs.append(obj)
        tasks.append(([nvcc, *NVCC_FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj], obj + ".log"))
    for src in ("fbf_params.cpp", "fbf_synth.cpp"):
        obj = os.path.join(build_dir, src.replace(".cpp", ".o"))
        objs.append(obj)
        tasks.append((["g++", *CXX_FLAGS, "-c", os.path.join(CSRC, src), "-o", obj], obj + ".log"))
    with cf.ThreadPoolExecutor(jobs) as ex:
        futs = [ex.submit(_run, cmd, log) for cmd, log in tasks]
        for f in futs:
            f.result()
    _check_inlined(tasks)
    tmp = lib + ".tmp"
    _run([nvcc, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-lpthread"],
         os.path.join(build_dir, "link.log"))
    os.replace(tmp, lib)
    if verbose:
        print(f"built {lib}")
    return lib


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--jobs", type=int, default=None)
    ap.add_argument("--out", default=None, help="dev: library path (default: the in-tree libfbf.so)")
    ap.add_argument("-D", dest="defines", action="append", default=[], help="dev: extra macro")
    ap.add_argument("--radius", type=int, default=None, help="dev: specialise one radius only")
    a = ap.parse_args()
    print(build(force=a.force, jobs=a.jobs, verbose=True, out=a.out, defines=a.defines, radius=a.radius))


if __name__ == "__main__":
    sys.exit(main())
