"""Build libfek.so (sm_100a) in-tree.

    python -m paper_1504_01023_b200.build_native [--force] [-j N]

The CUDA library is compiled per translation unit in parallel (fek_abi.cu plus
one TU per dtype x element x problem in csrc/cases/) and linked with a static
CUDA runtime, so the resulting ``paper_1504_01023_b200/libfek.so`` travels to
the GPU box with the repository snapshot and needs only the driver there.

Flags: ``-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20
--fmad=false`` -- no implicit FMA contraction, so the explicit ``fma()`` calls
fix one instruction sequence per element (bitwise layout/GPU-count
independence).
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "fek")
LIB = os.path.join(PKG, "libfek.so")
INCLUDE = os.path.join(ROOT, "include")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++20", "--fmad=false",
    "-Xptxas", "-v", "-Xcompiler", "-fPIC,-O2",
    "-I", INCLUDE,
]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _sources() -> list[str]:
    return [os.path.join(CSRC, n) for n in ("fek_abi.cu", "fek_mesh.cu", "fek_layout.cu")] + sorted(
        glob.glob(os.path.join(CSRC, "cases", "*.cu")))


def _headers() -> list[str]:
    return glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + [
        os.path.join(INCLUDE, "fek.h")]


def _obj_for(src: str) -> str:
    rel = os.path.relpath(src, CSRC).replace(os.sep, "_")
    return os.path.join(BUILD, rel[:-3] + ".o")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _compile(src: str, obj: str) -> tuple[str, str]:
    cmd = [_nvcc(), *NVCC_FLAGS, "-c", src, "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = res.stdout + res.stderr
    with open(obj + ".log", "w") as fh:
        fh.write(" ".join(cmd) + "\n" + log)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{log[-4000:]}")
    return src, log


def build_library(force: bool = False, jobs: int | None = None, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = _headers()
    todo = []
    for src in _sources():
        obj = _obj_for(src)
        if force or _stale(obj, [src, *headers]):
            todo.append((src, obj))
    if todo:
        jobs = jobs or min(len(todo), os.cpu_count() or 1)
        with cf.ThreadPoolExecutor(max_workers=jobs) as pool:
            for src, log in pool.map(lambda a: _compile(*a), todo):
                if verbose:
                    print(f"compiled {os.path.relpath(src, ROOT)}", file=sys.stderr)
    objs = [_obj_for(s) for s in _sources()]
    if force or todo or _stale(LIB, objs):
        tmp = LIB + ".tmp"
        cmd = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
               "-Xcompiler", "-fPIC", *objs, "-o", tmp]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stdout}{res.stderr}")
        os.replace(tmp, LIB)
    return LIB


def register_report() -> list[tuple[str, int, int, int]]:
    """(kernel, registers, spill-store bytes, spill-load bytes) from the ptxas logs."""
    import re

    rows = []
    pat = re.compile(r"Compiling entry function '(\S+)' for 'sm_100a'\n.*?Function properties for \S+\n\s*"
                     r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads\n"
                     r"ptxas info\s+: Used (\d+) registers", re.S)
    for log in glob.glob(os.path.join(BUILD, "*.log")):
        text = open(log).read()
        for name, _stack, ss, sl, regs in pat.findall(text):
            rows.append((name, int(regs), int(ss), int(sl)))
    return rows


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", "--jobs", type=int, default=None)
    ap.add_argument("--registers", action="store_true", help="print per-kernel register/spill report")
    args = ap.parse_args(argv)
    lib = build_library(force=args.force, jobs=args.jobs, verbose=True)
    print(lib)
    if args.registers:
        for name, regs, ss, sl in sorted(register_report()):
            print(f"{regs:4d} regs  spill {ss:4d}/{sl:4d}  {name}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
