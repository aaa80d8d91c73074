"""Helpers for the GPU parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np
import torch

KIND_DT = {"herm_d": (np.float64, torch.float64), "herm_z": (np.complex128, torch.complex128),
           "lu_z": (np.complex128, torch.complex128), "herm_s": (np.float32, torch.float32),
           "lu_c": (np.complex64, torch.complex64)}
FACTOR_TOL = 1e-9     # north_star: factor entries within 1e-9 relative to max|K|
LOGLIK_TOL = 1e-10    # north_star: log-likelihood within 1e-10 relative


def to_device(K: np.ndarray, kind: str, ld: int | None = None) -> torch.Tensor:
    """Column-major device storage (cols, ld) of the natural matrix K."""
    npdt, tdt = KIND_DT[kind]
    n = K.shape[0]
    ld = ld or max(n, 1)
    buf = np.zeros((max(n, 1), ld), dtype=npdt)
    buf[:n, :n] = np.asarray(K, dtype=npdt).T
    return torch.from_numpy(buf).to("cuda")


def from_device(Kc: torch.Tensor, n: int) -> np.ndarray:
    return Kc.cpu().numpy()[:n, :n].T.copy()


def compare_masks(gpu_mask: np.ndarray, o) -> int:
    """Bit-exact where the oracle saw no tie; else compare the prefix before the first tie.
    Returns the number of compared decisions."""
    gpu_mask = np.asarray(gpu_mask).astype(np.uint8)
    if o.n_ties == 0:
        assert np.array_equal(gpu_mask, o.mask), f"mask mismatch at {np.flatnonzero(gpu_mask != o.mask)[:10]}"
        return len(o.mask)
    k = o.first_tie
    assert np.array_equal(gpu_mask[:k], o.mask[:k])
    return k


def factor_part(F: np.ndarray, kind: str) -> np.ndarray:
    """The entries the sampler owns: lower triangle for Hermitian kinds, all for LU."""
    if kind in ("lu_z", "lu_c"):
        return F
    return np.tril(F)


def assert_factor_close(Fg: np.ndarray, Fo: np.ndarray, K: np.ndarray, kind: str):
    scale = (float(np.max(np.abs(K))) if K.size else 0.0) or 1.0
    d = np.max(np.abs(factor_part(Fg, kind) - factor_part(Fo, kind))) if Fg.size else 0.0
    assert d <= FACTOR_TOL * scale, f"factor max diff {d:.3e} > {FACTOR_TOL * scale:.3e}"
    return d


def assert_loglik_close(lg: float, lo: float):
    assert abs(lg - lo) <= LOGLIK_TOL * abs(lo) + 1e-12, f"loglik {lg!r} vs oracle {lo!r}"


def check_decisions(mask: np.ndarray, pivots: np.ndarray, seed: int, b: int, oracle_mod, tie_tol: float = 1e-9):
    """Every decision of a sample of ANY size against the oracle's uniforms (Listing 1 decision,
    PAPER.md:435-440): the pre-decision pivot is recovered from the returned factor as
    p_j = Re(final pivot_j) + (1 - mask_j) (the sampler subtracts 1 exactly when it drops j), u_j is
    recomputed with the ORACLE's Philox, and mask_j == (u_j <= p_j) must hold wherever
    |u_j - p_j| > tie_tol.  Returns the number of ties (pivots within tie_tol).  Together with a
    factor residual check (L D L^H = K - 1_{Y^c}) this pins the whole sample, not only a prefix."""
    mask = np.asarray(mask).astype(np.int64)
    p = np.asarray(pivots).real.astype(np.float64) + (1 - mask)
    u = np.array([oracle_mod.uniform(seed, j, b) for j in range(len(mask))])
    tie = np.abs(u - p) <= tie_tol
    want = (u <= p).astype(np.int64)
    bad = np.flatnonzero((want != mask) & ~tie)
    assert bad.size == 0, f"decisions inconsistent with the oracle's uniforms at {bad[:10]}"
    return int(tie.sum())
