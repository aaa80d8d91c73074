"""Builds and runs tests/tools/curand_philox_kat.cu: curand's Philox4x32-10 on the host
(a library routine) -- the independent pin for both Philox implementations."""
import os
import shutil
import subprocess
import tempfile

import pytest

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tools", "curand_philox_kat.cu")
_BIN = None


def curand_philox(rows):
    """rows: list of (c0, c1, c2, c3, k0, k1) -> list of 4-tuples from curand."""
    global _BIN
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available to build the curand KAT tool")
    if _BIN is None:
        d = tempfile.mkdtemp(prefix="dppkat")
        _BIN = os.path.join(d, "kat")
        subprocess.check_call([nvcc, "-Wno-deprecated-gpu-targets", "-o", _BIN, _SRC],
                              stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    inp = "\n".join(" ".join(str(int(v) & 0xFFFFFFFF) for v in r) for r in rows) + "\n"
    out = subprocess.run([_BIN], input=inp, capture_output=True, text=True, check=True).stdout
    return [tuple(int(x) for x in line.split()) for line in out.strip().splitlines()]
