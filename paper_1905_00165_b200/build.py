"""Builds libdpp_b200.so in-tree: nvcc for sm_100a only (no other architectures, no JIT)."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libdpp_b200.so")
SOURCES = ["diag.cu", "diag_rl.cu", "update.cu", "update_ws.cu", "update_simt.cu", "update_tc32.cu", "next_tile.cu", "elementary.cu", "lensemble.cu", "driver.cu", "dist.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for c in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found: cannot build the sm_100a library")


def _nccl_flags():
    for d in ("/usr/lib/x86_64-linux-gnu", "/usr/lib64", "/usr/local/lib"):
        if os.path.exists(os.path.join(d, "libnccl.so")) or os.path.exists(os.path.join(d, "libnccl.so.2")):
            inc = "/usr/include" if os.path.exists("/usr/include/nccl.h") else None
            return ([f"-I{inc}"] if inc else []), [f"-L{d}", "-lnccl"]
    raise RuntimeError("NCCL headers/library not found")


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    nvcc = _nvcc()
    inc_nccl, lib_nccl = _nccl_flags()
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
        os.path.join(os.path.dirname(HERE), "include", "dpp.h"), __file__]
    newest_dep = max(os.path.getmtime(p) for p in deps)
    objs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src.replace(".cu", ".o"))
        objs.append(o)
        if force or not os.path.exists(o) or os.path.getmtime(o) < newest_dep:
            cmd = [nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                   "-I" + os.path.join(os.path.dirname(HERE), "include"), *inc_nccl, "-c", s, "-o", o]
            r = subprocess.run(cmd, capture_output=True, text=True)
            with open(o + ".ptxas.txt", "w") as f:  # (compile times dropped: the log stays diff-stable)
                f.write("".join(l for l in (r.stdout + r.stderr).splitlines(True) if "Compile time" not in l))
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {src}")
            if verbose:
                sys.stderr.write(r.stderr)
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [nvcc, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, *lib_nccl,
               "-Xlinker", "-rpath=/usr/lib/x86_64-linux-gnu"]
        subprocess.check_call(cmd)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
