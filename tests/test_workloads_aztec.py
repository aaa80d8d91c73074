"""Balanced-gauge Kenyon kernel of the Aztec diamond (BASELINE.json configs[2]; reading R13).

Harness checks (no GPU): the balanced kernel M' = D M D^{-1} (Prop. 2) equals
the plain-gauge Kenyon kernel conjugated by the power-of-two gauge where the plain gauge is
accurate (d <= 20), and at larger d it keeps the invariants every Kenyon kernel has:
  * diag M'_ii = P(e_i in the tiling) is real and in [0, 1];
  * trace M' = d(d+1) (the number of dominoes);
  * for each black square b, sum of M'_ii over its edges = (K' K'^{-1})(b, b) = 1;
and the oracle sampling it draws perfect tilings with the paper's likelihood.
"""
import json
import os

import numpy as np
import pytest

import workloads as W

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_pins.json")))


def _invariants(d, M, edges):
    n = len(edges)
    assert M.shape == (n, n) and n == 4 * d * d
    dg = np.diag(M)
    assert np.max(np.abs(dg.imag)) <= 1e-12
    assert dg.real.min() >= -1e-12 and dg.real.max() <= 1 + 1e-12
    assert abs(dg.real.sum() - d * (d + 1)) <= 1e-9 * d * d
    per_black = np.zeros(d * (d + 1))
    np.add.at(per_black, np.array([e[0] for e in edges]), dg.real)
    assert np.max(np.abs(per_black - 1.0)) <= 1e-12


@pytest.mark.parametrize("d", [10, 20])
def test_balanced_equals_plain_gauge_conjugated(d):
    M, info = W.aztec_kernel_balanced(d, storage="natural", return_info=True)
    M = M.numpy()
    M0 = W.aztec_kernel(d)
    a = info["a_black"]
    Dv = np.array([2.0 ** a[e[0]] for e in info["edges"]])
    M1 = Dv[:, None] * M0 / Dv[None, :]
    # the plain gauge's own inverse error grows with d (~4e-12 at d = 20)
    assert np.max(np.abs(M1 - M)) <= (1e-12 if d == 10 else 1e-9)
    assert np.max(np.abs(M)) <= 1.0 + 1e-12
    _invariants(d, M, info["edges"])


def test_balanced_invariants_d30():
    M, info = W.aztec_kernel_balanced(30, storage="natural", return_info=True)
    for st in info["steps"]:
        assert st["inverse_residual"] <= 1e-13
    _invariants(30, M.numpy(), info["edges"])


def test_colmajor_storage_is_transpose():
    T = W.aztec_kernel_balanced(6).numpy()
    M = W.aztec_kernel_balanced(6, storage="natural").numpy()
    assert np.array_equal(T, M.T)


def test_oracle_on_balanced_kernel_d10(oracle_mod):
    """The balanced kernel defines the same DPP: oracle samples are perfect tilings with
    likelihood e^{-38.1231}, = -55 ln 2 in closed form."""
    M = W.aztec_kernel_balanced(10, storage="natural").numpy()
    want = -55 * np.log(2.0)
    for b in range(3):
        r = oracle_mod.sample_lu_z(np.asfortranarray(M), 0, b)
        assert W.is_aztec_tiling(10, r.mask)
        assert abs(r.loglik - want) <= 1e-10 * abs(want)
        assert round(r.loglik, 4) == GOLD["aztec_d10_loglik"]["value"]
