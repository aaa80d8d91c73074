"""CPU checks of the C-ABI library: it builds for sm_100a, loads, exports every symbol
include/dpp.h declares, and its host-only helpers behave (no compute without a GPU)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libpath():
    from paper_1905_00165_b200 import build
    return build.build()


def _declared():
    src = open(os.path.join(ROOT, "include", "dpp.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const char\*|int64_t|size_t|int)\s+(dpp_\w+)\s*\(", src, re.M)))


def test_exports_every_declared_symbol(libpath):
    names = _declared()
    assert len(names) >= 18
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (dpp_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    import paper_1905_00165_b200 as dpp
    assert sorted(dpp.EXPORTS) == names


def test_sm100a_only(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_tensor_core_and_async_copy_in_sass(libpath):
    """The update kernels are on the FP64 tensor path (DMMA): the warp-specialized one fed by TMA
    bulk copies (UBLKCP) behind mbarriers (SYNCS), the fallback by cp.async (LDGSTS)."""
    out = subprocess.run(["cuobjdump", "-sass", libpath], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in out
    assert "UBLKCP" in out and "SYNCS" in out
    assert "LDGSTS" in out
    # the fp32 updates on the 5th-generation tensor cores: tcgen05.mma (UTCHMMA), tcgen05.ld (LDTM)
    assert "UTCHMMA" in out and "LDTM" in out


def test_host_helpers():
    import paper_1905_00165_b200 as dpp
    assert dpp.dpp_version().startswith("dpp-b200")
    # in-place calls need the per-sample state, the tile operators, D1 and the panel buffers
    # (W21 = L21 D1, or U12^T for LU, in two group buffers of G = 3 panels: ldk x nb each) -- no n x n
    # buffer
    ws = dpp.dpp_workspace_bytes(dpp.DPP_OP_HERM_D, 1, 16384)
    assert 6 * 16384 * 128 * 8 < ws < 6 * 16384 * 128 * 8 + 400_000
    ws = dpp.dpp_workspace_bytes(dpp.DPP_OP_LU_Z, 1, 1000)
    assert 6 * 1008 * 64 * 16 + 2 * 64 * 64 * 16 < ws < 6 * 1008 * 64 * 16 + 400_000
    # the fp32 sampler's tensor-core updates add two scratch regions for their packed operands
    assert dpp.dpp_workspace_bytes(dpp.DPP_OP_HERM_S, 1, 4096) > dpp.dpp_workspace_bytes(
        dpp.DPP_OP_HERM_S, 1, 4096, dpp.make_opts(flags=dpp.DPP_FLAG_FP32_SIMT))
    assert dpp.dpp_workspace_bytes(dpp.DPP_OP_HERM_D | dpp.DPP_OP_BATCHED, 4, 100) >= 4 * 112 * 100 * 8
    assert dpp.dpp_workspace_bytes(dpp.DPP_OP_HERM_D, 1, 10, dpp.make_opts(nb=48)) == 0
    for n, nb, P in [(1000, 128, 3), (16384, 128, 8), (65536, 128, 8), (100, 128, 4), (0, 128, 2)]:
        cols = [dpp.dpp_bcc_local_cols(n, nb, P, r) for r in range(P)]
        assert sum(cols) == n
        assert max(cols) - min(cols) <= nb
    assert dpp.dpp_bcc_local_cols(10, 128, 2, 2) == -1
    assert dpp._lib.dpp_strerror(-2).decode().startswith("workspace")
