"""CPU oracle for the factorization-based DPP sampler -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_1905_00165_b200`` never imports it and shares no code with it.

Thin ctypes marshalling over ``dpp_oracle.c`` (plain C, fp64, one thread, no
BLAS), which follows Listing 1 of arXiv 1905.00165 step by
step; see the header of that file for the readings R1-R8 it implements.

Pinned by ``tests/test_oracle_*.py`` (-m "not gpu"):
  * Philox:    KAT against curand's ``curand_Philox4x32_10`` (library routine).
  * decisions: K = diag(p) closed form; K = 0, K = I.
  * law:       brute-force subset frequencies vs |det(K - 1_{S^c})|.
  * structure: projection cardinality = rank, UST spanning
               trees with loglik -ln tau(G), Aztec tilings with
               loglik -d(d+1)/2 ln 2.
  * factor:    L D L^H = K - 1_{Y^c}, L U = K - 1_{Y^c}; loglik = ln|det| (slogdet).
  * prefix:    decisions on K[:m,:m] = first m decisions on K (loop invariant,
               PAPER.md:402-405).
  * fp32 (reading R19): diag(p) closed form in fp32, brute-force law of the
               fp32 kernel, agreement with the fp64 oracle within fp32 rounding, UST and
               Aztec structure (tests/test_oracle_fp32.py).
  * elementary sampler (Listing 2, reading R20; tests/test_oracle_elementary.py): cardinality k,
               loglik = ln det(K_Y) (slogdet), factor = Cholesky of K_Y, brute-force law,
               marginals, UST trees.
  * L-ensemble conversion K = I - (L+I)^{-1} (tests/test_oracle_lensemble.py):
               eigenvalue map lambda / (1 + lambda), special cases, and the DPP law of the
               converted kernel vs the L-ensemble's det(L_S) / det(L + I) by brute force.
  * greedy MAP: K = diag(p) closed form; every decision takes the
               branch whose leading-principal-minor probability |det| is larger
               (numpy det, brute force over both branches at every pivot).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dpp_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

HERM_D, HERM_Z, LU_Z, HERM_S, LU_C = 0, 1, 2, 3, 4
TIE_TOL = 1e-9
RANGE_TOL = 1e-8


class _Info(ctypes.Structure):
    _fields_ = [
        ("n_kept", ctypes.c_int32),
        ("n_ties", ctypes.c_int32),
        ("first_tie", ctypes.c_int32),
        ("n_out_of_range", ctypes.c_int32),
        ("min_abs_pivot", ctypes.c_double),
        ("max_abs_imag_pivot", ctypes.c_double),
    ]


@dataclass
class OracleResult:
    mask: np.ndarray          # uint8[n], 1 = kept
    loglik: float
    factor: np.ndarray        # in-place factor of K - 1_{Y^c} (column-major semantics)
    n_kept: int
    n_ties: int
    first_tie: int
    n_out_of_range: int
    min_abs_pivot: float
    max_abs_imag_pivot: float


def build(force: bool = False) -> str:
    """Compile the oracle (gcc -O2 -ffp-contract=off, one thread, no BLAS)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-std=c11", "-shared", "-fPIC",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        for name in ("oracle_sample_herm_d", "oracle_sample_herm_z", "oracle_sample_lu_z",
                     "oracle_sample_herm_s", "oracle_sample_lu_c"):
            f = getattr(_lib, name)
            f.restype = ctypes.c_int
            f.argtypes = [ctypes.c_int64, P, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64, P,
                          ctypes.c_double, ctypes.c_double, P, P, P]
        for name in ("oracle_map_herm_d", "oracle_map_herm_z", "oracle_map_lu_z"):
            f = getattr(_lib, name)
            f.restype = ctypes.c_int
            f.argtypes = [ctypes.c_int64, P, ctypes.c_int64, P, ctypes.c_double, ctypes.c_double, P, P, P]
        _lib.oracle_elementary_herm_d.restype = ctypes.c_int
        _lib.oracle_elementary_herm_d.argtypes = [ctypes.c_int64, ctypes.c_int64, P, ctypes.c_int64, ctypes.c_uint64,
                                                  ctypes.c_uint64, ctypes.c_double, P, P, P, P, P]
        _lib.oracle_uniform.restype = ctypes.c_double
        _lib.oracle_uniform.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64]
        _lib.oracle_philox4x32_10.restype = None
        _lib.oracle_philox4x32_10.argtypes = [P, P, P]
        _lib.oracle_sample_many.restype = ctypes.c_int
        _lib.oracle_sample_many.argtypes = [ctypes.c_int, ctypes.c_int64, P, ctypes.c_int64,
                                            ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, P, P]
    return _lib


def philox4x32_10(ctr, key) -> tuple:
    c = (ctypes.c_uint32 * 4)(*[int(v) & 0xFFFFFFFF for v in ctr])
    k = (ctypes.c_uint32 * 2)(*[int(v) & 0xFFFFFFFF for v in key])
    o = (ctypes.c_uint32 * 4)()
    lib().oracle_philox4x32_10(c, k, o)
    return tuple(int(v) for v in o)


def uniform(seed: int, j: int, b: int = 0) -> float:
    return float(lib().oracle_uniform(seed, j, b))


def _as_colmajor(K: np.ndarray, kind: int) -> np.ndarray:
    dt = {HERM_D: np.float64, HERM_Z: np.complex128, LU_Z: np.complex128, HERM_S: np.float32,
          LU_C: np.complex64}[kind]
    return np.array(K, dtype=dt, order="F", copy=True)


def sample(kind: int, K: np.ndarray, seed: int = 0, b: int = 0, forced=None,
           tie_tol: float = TIE_TOL, range_tol: float = RANGE_TOL) -> OracleResult:
    """One sample of DPP(K) by Listing 1 (kind = HERM_D | HERM_Z | LU_Z)."""
    A = _as_colmajor(K, kind)
    n = A.shape[0]
    assert A.shape == (n, n)
    mask = np.zeros(max(n, 1), dtype=np.uint8)
    ll = ctypes.c_double(0.0)
    info = _Info()
    fptr = None
    if forced is not None:
        forced = np.ascontiguousarray(np.asarray(forced, dtype=np.uint8))
        assert forced.shape == (n,)
        fptr = forced.ctypes.data
    fn = {HERM_D: lib().oracle_sample_herm_d, HERM_Z: lib().oracle_sample_herm_z,
          LU_Z: lib().oracle_sample_lu_z, HERM_S: lib().oracle_sample_herm_s,
          LU_C: lib().oracle_sample_lu_c}[kind]
    rc = fn(n, A.ctypes.data, max(n, 1), seed, b, fptr, tie_tol, range_tol,
            mask.ctypes.data, ctypes.byref(ll), ctypes.byref(info))
    if rc != 0:
        raise RuntimeError(f"oracle returned {rc}")
    return OracleResult(mask[:n].copy(), ll.value, A, info.n_kept, info.n_ties, info.first_tie,
                        info.n_out_of_range, info.min_abs_pivot, info.max_abs_imag_pivot)


def greedy_map(kind: int, K: np.ndarray, forced=None, tie_tol: float = TIE_TOL,
               range_tol: float = RANGE_TOL) -> OracleResult:
    """Greedy maximum-likelihood inference (reading R18): Listing 1 with each
    Bernoulli draw replaced by the more probable branch, keep iff Re p >= 1/2."""
    A = _as_colmajor(K, kind)
    n = A.shape[0]
    assert A.shape == (n, n)
    mask = np.zeros(max(n, 1), dtype=np.uint8)
    ll = ctypes.c_double(0.0)
    info = _Info()
    fptr = None
    if forced is not None:
        forced = np.ascontiguousarray(np.asarray(forced, dtype=np.uint8))
        fptr = forced.ctypes.data
    fn = {HERM_D: lib().oracle_map_herm_d, HERM_Z: lib().oracle_map_herm_z, LU_Z: lib().oracle_map_lu_z}[kind]
    rc = fn(n, A.ctypes.data, max(n, 1), fptr, tie_tol, range_tol, mask.ctypes.data, ctypes.byref(ll),
            ctypes.byref(info))
    if rc != 0:
        raise RuntimeError(f"oracle returned {rc}")
    return OracleResult(mask[:n].copy(), ll.value, A, info.n_kept, info.n_ties, info.first_tie,
                        info.n_out_of_range, info.min_abs_pivot, info.max_abs_imag_pivot)


@dataclass
class ElementaryResult:
    order: np.ndarray      # int64[k]: chosen items (original indices) in pivot order
    loglik: float          # sum_j ln d_{t_j} = ln det(K_Y)
    L: np.ndarray          # n x k factor, rows by original index (L_Y = Cholesky factor of K_Y)
    n_ties: int
    first_tie: int

    @property
    def mask(self):
        m = np.zeros(self.L.shape[0], dtype=np.uint8)
        m[self.order] = 1
        return m


def elementary_herm_d(K: np.ndarray, k: int, seed: int = 0, b: int = 0, tie_tol: float = 1e-12) -> ElementaryResult:
    """Listing 2 for a real rank-k projection K, reading R20."""
    A = np.array(K, dtype=np.float64, order="F", copy=True)
    n = A.shape[0]
    order = np.zeros(max(k, 1), dtype=np.int64)
    L = np.zeros((n, max(k, 1)), dtype=np.float64, order="F")
    ll = ctypes.c_double(0.0)
    nt, ft = ctypes.c_int32(0), ctypes.c_int32(-1)
    rc = lib().oracle_elementary_herm_d(n, k, A.ctypes.data, max(n, 1), seed, b, tie_tol, order.ctypes.data,
                                        L.ctypes.data, ctypes.byref(ll), ctypes.byref(nt), ctypes.byref(ft))
    if rc != 0:
        raise RuntimeError(f"oracle returned {rc}")
    return ElementaryResult(order[:k].copy(), ll.value, L[:, :k], nt.value, ft.value)


def lensemble_to_marginal(L: np.ndarray):
    """K = I - (L + I)^{-1} (Gillenwater 2014) for a Hermitian PSD L-ensemble
    kernel -- the plain definition with a library inverse (fp64), plus ln det(L + I).  Not the
    paper's algorithm (which the GPU path follows: factorization, triangular inverse, product)."""
    L = np.asarray(L)
    n = L.shape[0]
    M = L + np.eye(n, dtype=L.dtype)
    K = np.eye(n, dtype=L.dtype) - np.linalg.inv(M)
    sign, logdet = np.linalg.slogdet(M)
    return K, float(logdet)


def sample_herm_d(K, seed=0, b=0, forced=None, **kw):
    return sample(HERM_D, K, seed, b, forced, **kw)


def sample_herm_z(K, seed=0, b=0, forced=None, **kw):
    return sample(HERM_Z, K, seed, b, forced, **kw)


def sample_lu_z(K, seed=0, b=0, forced=None, **kw):
    return sample(LU_Z, K, seed, b, forced, **kw)


def sample_herm_s(K, seed=0, b=0, forced=None, **kw):
    """Single-precision real symmetric sampler (reading R19): fp32 factorization, fp64 decisions
    against the fp32 pivot, fp64 log-likelihood accumulation."""
    return sample(HERM_S, K, seed, b, forced, **kw)


def sample_lu_c(K, seed=0, b=0, forced=None, **kw):
    """Single-precision complex non-Hermitian LU sampler (reading R19)."""
    return sample(LU_C, K, seed, b, forced, **kw)


def sample_many(kind: int, K: np.ndarray, seed: int, b0: int, batch: int):
    """Masks (batch x n, uint8) and logliks (batch) of samples b0..b0+batch-1."""
    A = _as_colmajor(K, kind)
    n = A.shape[0]
    masks = np.zeros((batch, max(n, 1)), dtype=np.uint8)
    lls = np.zeros(batch, dtype=np.float64)
    rc = lib().oracle_sample_many(kind, n, A.ctypes.data, max(n, 1), seed, b0, batch,
                                  masks.ctypes.data, lls.ctypes.data)
    if rc != 0:
        raise RuntimeError(f"oracle returned {rc}")
    return masks[:, :n], lls
