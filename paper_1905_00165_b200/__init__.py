"""B200-native factorization-based DPP sampler (arXiv 1905.00165) -- Python binding.

Argument marshalling only: every step of the sampler runs in the sm_100a kernels of
``libdpp_b200.so`` behind the C ABI declared in ``include/dpp.h``.  There is no CPU
fallback: importing this package raises if the library is missing, and every call
raises if the library returns an error.

Storage convention: matrices are column-major.  A torch tensor ``Kc`` of shape
(cols, ld) (row-major, contiguous) holds the column-major matrix K with leading
dimension ld: ``Kc[l, i] == K[i, l]``.  ``colmajor(K)`` converts a natural (row-major
indexed) matrix; for Hermitian K, colmajor(K) == K.conj().
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdpp_b200.so")

DPP_OP_HERM_D, DPP_OP_HERM_Z, DPP_OP_LU_Z, DPP_OP_HERM_S, DPP_OP_LU_C = 0, 1, 2, 3, 4
DPP_OP_BATCHED, DPP_OP_HOST = 0x10, 0x20
INFO_BYTES = 32

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1905_00165_b200.build` "
                      "(there is no CPU fallback)")


class dpp_opts_t(ctypes.Structure):
    _fields_ = [("nb", ctypes.c_int32), ("lookahead", ctypes.c_int32), ("tie_tol", ctypes.c_double),
                ("range_tol", ctypes.c_double), ("forced", ctypes.c_void_p), ("batch_chunk", ctypes.c_int64),
                ("group", ctypes.c_int32), ("flags", ctypes.c_uint32), ("group_min_rows", ctypes.c_int64)]


DPP_FLAG_GENERIC_UPDATE = 1
DPP_FLAG_FP32_SIMT = 2
DPP_FLAG_NO_SPLIT_CHAIN = 4


class dpp_info_t(ctypes.Structure):
    _fields_ = [("n_kept", ctypes.c_int32), ("n_ties", ctypes.c_int32), ("first_tie", ctypes.c_int32),
                ("n_out_of_range", ctypes.c_int32), ("min_abs_pivot", ctypes.c_double),
                ("max_abs_imag_pivot", ctypes.c_double)]


_lib = ctypes.CDLL(LIB_PATH)
_P, _I64, _U64, _SZ = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_size_t


def _sig(name, res, args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = args
    return f


_sig("dpp_workspace_bytes", _SZ, [ctypes.c_int, _I64, _I64, _P])
for _n in ("dpp_sample_herm_d", "dpp_sample_herm_z", "dpp_sample_lu_z", "dpp_sample_herm_s", "dpp_sample_lu_c"):
    _sig(_n, ctypes.c_int, [_I64, _P, _I64, _U64, _P, _P, _P, _P, _P, _SZ, _P])
for _n in ("dpp_map_herm_d", "dpp_map_herm_z", "dpp_map_lu_z"):
    _sig(_n, ctypes.c_int, [_I64, _P, _I64, _P, _P, _P, _P, _P, _SZ, _P])
for _n in ("dpp_sample_herm_d_batched", "dpp_sample_herm_z_batched", "dpp_sample_lu_z_batched",
           "dpp_sample_herm_s_batched", "dpp_sample_lu_c_batched", "dpp_elementary_workspace_bytes",
           "dpp_elementary_herm_d", "dpp_lensemble_workspace_bytes", "dpp_lensemble_to_marginal_d",
           "dpp_lensemble_to_marginal_z",
           "dpp_sample_herm_d_host", "dpp_sample_herm_z_host", "dpp_sample_lu_z_host",
           "dpp_sample_herm_d_host_async", "dpp_sample_herm_z_host_async", "dpp_sample_lu_z_host_async"):
    _sig(_n, ctypes.c_int, [_I64, _I64, _P, _I64, _I64, _U64, _U64, _P, _P, _P, _P, _P, _SZ, _P])
_sig("dpp_elementary_workspace_bytes", _SZ, [_I64, _I64, _I64])
_sig("dpp_lensemble_workspace_bytes", _SZ, [ctypes.c_int, _I64])
for _n in ("dpp_lensemble_to_marginal_d", "dpp_lensemble_to_marginal_z"):
    _sig(_n, ctypes.c_int, [_I64, _P, _I64, _P, _P, _SZ, _P])
_sig("dpp_elementary_herm_d", ctypes.c_int, [_I64, _I64, _I64, _P, _I64, _U64, _U64, _P, _P, _P, _P, _SZ, _P])
_sig("dpp_philox_uniforms", ctypes.c_int, [_U64, _U64, _U64, _I64, _P, _P])
_sig("dpp_comm_init", ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_P)])
_sig("dpp_comm_init_local", ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_P)])
_sig("dpp_comm_destroy", ctypes.c_int, [_P])
_sig("dpp_dist_message_bytes", _I64, [ctypes.c_int, _I64, ctypes.c_int, _I64])
for _n in ("dpp_sample_herm_d_dist_local", "dpp_sample_herm_z_dist_local"):
    _sig(_n, ctypes.c_int, [_P, _I64, _P, _I64, _U64, _P, _P, _P, _P, _P, _SZ, _P])
_sig("dpp_bcc_local_cols", _I64, [_I64, ctypes.c_int32, ctypes.c_int, ctypes.c_int])
_sig("dpp_dist_workspace_bytes", _SZ, [ctypes.c_int, _I64, ctypes.c_int, _P])
for _n in ("dpp_sample_herm_d_dist", "dpp_sample_herm_z_dist"):
    _sig(_n, ctypes.c_int, [_P, _I64, _P, _I64, _U64, _P, _P, _P, _P, _P, _SZ, _P])
class dpp_profile_t(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_int64 * 5), ("ms", ctypes.c_double * 5), ("flops", ctypes.c_double * 5),
                ("ms_union", ctypes.c_double * 5), ("top_flops", ctypes.c_double * 5),
                ("top_ms", ctypes.c_double * 5)]


_sig("dpp_profile_begin", ctypes.c_int, [])
_sig("dpp_profile_begin_stages", ctypes.c_int, [ctypes.c_uint])
_sig("dpp_profile_end", ctypes.c_int, [ctypes.POINTER(dpp_profile_t)])
_sig("dpp_profile_end_records", ctypes.c_int, [ctypes.POINTER(dpp_profile_t), _P, _I64, ctypes.POINTER(_I64)])
_sig("dpp_probe_update_d", ctypes.c_int, [_I64, ctypes.c_int32, _P, _P, _I64, _P, _I64, ctypes.POINTER(ctypes.c_float), _P])
_sig("dpp_strerror", ctypes.c_char_p, [ctypes.c_int])
_sig("dpp_version", ctypes.c_char_p, [])

EXPORTS = ["dpp_workspace_bytes", "dpp_sample_herm_d", "dpp_sample_herm_z", "dpp_sample_lu_z",
           "dpp_map_herm_d", "dpp_map_herm_z", "dpp_map_lu_z", "dpp_sample_herm_s", "dpp_sample_lu_c",
           "dpp_sample_herm_s_batched", "dpp_sample_lu_c_batched", "dpp_elementary_workspace_bytes",
           "dpp_elementary_herm_d", "dpp_lensemble_workspace_bytes", "dpp_lensemble_to_marginal_d",
           "dpp_lensemble_to_marginal_z",
           "dpp_sample_herm_d_batched", "dpp_sample_herm_z_batched", "dpp_sample_lu_z_batched",
           "dpp_sample_herm_d_host_async", "dpp_sample_herm_z_host_async", "dpp_sample_lu_z_host_async",
           "dpp_sample_herm_d_host", "dpp_sample_herm_z_host", "dpp_sample_lu_z_host",
           "dpp_philox_uniforms", "dpp_comm_init", "dpp_comm_init_local", "dpp_comm_destroy", "dpp_bcc_local_cols",
           "dpp_dist_workspace_bytes", "dpp_dist_message_bytes", "dpp_sample_herm_d_dist", "dpp_sample_herm_z_dist",
           "dpp_sample_herm_d_dist_local", "dpp_sample_herm_z_dist_local", "dpp_profile_begin", "dpp_profile_begin_stages", "dpp_profile_end", "dpp_profile_end_records", "dpp_probe_update_d",
           "dpp_strerror", "dpp_version"]


class DppError(RuntimeError):
    pass


def _check(rc: int):
    if rc != 0:
        raise DppError(f"dpp error {rc}: {_lib.dpp_strerror(rc).decode()}")


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _stream(stream):
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def make_opts(nb=0, lookahead=1, tie_tol=0.0, range_tol=0.0, forced=None, batch_chunk=0, group=0, flags=0,
              group_min_rows=0):
    """dpp_opts_t (include/dpp.h); group_min_rows < 0 groups trailing updates at every size."""
    o = dpp_opts_t()
    o.nb, o.lookahead, o.tie_tol, o.range_tol = nb, lookahead, tie_tol, range_tol
    o.forced = _ptr(forced)
    o.batch_chunk = batch_chunk
    o.group, o.flags, o.group_min_rows = group, flags, group_min_rows
    return o


def _optp(opts):
    return ctypes.byref(opts) if opts is not None else None


# ------------------------------------------------------------------ thin C-ABI mirrors
def dpp_workspace_bytes(op: int, batch: int, n: int, opts=None) -> int:
    return int(_lib.dpp_workspace_bytes(op, batch, n, _optp(opts)))


def dpp_sample_herm_d(n, K, ld, seed, mask, loglik, info=None, opts=None, work=None, work_bytes=None, stream=None):
    _check(_lib.dpp_sample_herm_d(n, _ptr(K), ld, seed, _ptr(mask), _ptr(loglik), _ptr(info), _optp(opts),
                                  _ptr(work), work_bytes if work_bytes is not None else work.numel(), _stream(stream)))


def dpp_sample_herm_z(n, K, ld, seed, mask, loglik, info=None, opts=None, work=None, work_bytes=None, stream=None):
    _check(_lib.dpp_sample_herm_z(n, _ptr(K), ld, seed, _ptr(mask), _ptr(loglik), _ptr(info), _optp(opts),
                                  _ptr(work), work_bytes if work_bytes is not None else work.numel(), _stream(stream)))


def dpp_sample_lu_z(n, K, ld, seed, mask, loglik, info=None, opts=None, work=None, work_bytes=None, stream=None):
    _check(_lib.dpp_sample_lu_z(n, _ptr(K), ld, seed, _ptr(mask), _ptr(loglik), _ptr(info), _optp(opts),
                                _ptr(work), work_bytes if work_bytes is not None else work.numel(), _stream(stream)))


def _map(name):
    fn = getattr(_lib, name)

    def call(n, K, ld, mask, loglik, info=None, opts=None, work=None, work_bytes=None, stream=None):
        _check(fn(n, _ptr(K), ld, _ptr(mask), _ptr(loglik), _ptr(info), _optp(opts), _ptr(work),
                  work_bytes if work_bytes is not None else work.numel(), _stream(stream)))
    call.__name__ = name
    return call


dpp_map_herm_d = _map("dpp_map_herm_d")
dpp_map_herm_z = _map("dpp_map_herm_z")
dpp_map_lu_z = _map("dpp_map_lu_z")


def dpp_sample_herm_s(n, K, ld, seed, mask, loglik, info=None, opts=None, work=None, work_bytes=None, stream=None):
    _check(_lib.dpp_sample_herm_s(n, _ptr(K), ld, seed, _ptr(mask), _ptr(loglik), _ptr(info), _optp(opts),
                                  _ptr(work), work_bytes if work_bytes is not None else work.numel(), _stream(stream)))


def dpp_sample_lu_c(n, K, ld, seed, mask, loglik, info=None, opts=None, work=None, work_bytes=None, stream=None):
    _check(_lib.dpp_sample_lu_c(n, _ptr(K), ld, seed, _ptr(mask), _ptr(loglik), _ptr(info), _optp(opts),
                                _ptr(work), work_bytes if work_bytes is not None else work.numel(), _stream(stream)))


def _batched(name):
    fn = getattr(_lib, name)

    def call(batch, n, K, ld, strideK, seed, b0, mask, loglik, info=None, opts=None, work=None, work_bytes=None,
             stream=None):
        _check(fn(batch, n, _ptr(K), ld, strideK, seed, b0, _ptr(mask), _ptr(loglik), _ptr(info), _optp(opts),
                  _ptr(work), work_bytes if work_bytes is not None else work.numel(), _stream(stream)))
    call.__name__ = name
    return call


dpp_sample_herm_d_batched = _batched("dpp_sample_herm_d_batched")
dpp_sample_herm_z_batched = _batched("dpp_sample_herm_z_batched")
dpp_sample_lu_z_batched = _batched("dpp_sample_lu_z_batched")
dpp_sample_herm_d_host = _batched("dpp_sample_herm_d_host")
dpp_sample_herm_z_host = _batched("dpp_sample_herm_z_host")
dpp_sample_lu_z_host = _batched("dpp_sample_lu_z_host")
dpp_sample_herm_d_host_async = _batched("dpp_sample_herm_d_host_async")
dpp_sample_herm_z_host_async = _batched("dpp_sample_herm_z_host_async")
dpp_sample_lu_z_host_async = _batched("dpp_sample_lu_z_host_async")
dpp_sample_herm_s_batched = _batched("dpp_sample_herm_s_batched")
dpp_sample_lu_c_batched = _batched("dpp_sample_lu_c_batched")


def dpp_elementary_workspace_bytes(batch, n, k) -> int:
    return int(_lib.dpp_elementary_workspace_bytes(batch, n, k))


def dpp_elementary_herm_d(batch, n, k, K, ld, seed, b0, order, loglik, ties=None, work=None, work_bytes=None,
                          stream=None):
    _check(_lib.dpp_elementary_herm_d(batch, n, k, _ptr(K), ld, seed, b0, _ptr(order), _ptr(loglik), _ptr(ties),
                                      _ptr(work), work_bytes if work_bytes is not None else work.numel(),
                                      _stream(stream)))


def elementary(Kc: torch.Tensor, k: int, batch: int = 1, seed: int = 0, b0: int = 0, work=None, stream=None):
    """Elementary DPP sampler (Listing 2) for a rank-k projection kernel in column-major storage
    Kc (n, ld): returns (order [batch, k] int64, loglik [batch], ties [batch, 2] int32)."""
    n, ld = Kc.shape[0], Kc.shape[1]
    dev = Kc.device
    order = torch.empty((batch, max(k, 1)), dtype=torch.int64, device=dev)
    ll = torch.empty(batch, dtype=torch.float64, device=dev)
    ties = torch.empty((batch, 2), dtype=torch.int32, device=dev)
    if work is None:
        work = torch.empty(max(dpp_elementary_workspace_bytes(batch, n, k), 256), dtype=torch.uint8, device=dev)
    dpp_elementary_herm_d(batch, n, k, Kc, ld, seed, b0, order, ll, ties, work, stream=stream)
    return order[:, :k], ll, ties


def dpp_lensemble_workspace_bytes(op, n) -> int:
    return int(_lib.dpp_lensemble_workspace_bytes(op, n))


def dpp_lensemble_to_marginal_d(n, A, ld, logdet=None, work=None, work_bytes=None, stream=None):
    _check(_lib.dpp_lensemble_to_marginal_d(n, _ptr(A), ld, _ptr(logdet), _ptr(work),
                                            work_bytes if work_bytes is not None else work.numel(), _stream(stream)))


def dpp_lensemble_to_marginal_z(n, A, ld, logdet=None, work=None, work_bytes=None, stream=None):
    _check(_lib.dpp_lensemble_to_marginal_z(n, _ptr(A), ld, _ptr(logdet), _ptr(work),
                                            work_bytes if work_bytes is not None else work.numel(), _stream(stream)))


def lensemble_to_marginal(Lc: torch.Tensor, work=None, stream=None):
    """K = I - (L + I)^{-1} in place on the lower triangle of the column-major storage Lc (n, ld),
    real (float64) or complex Hermitian (complex128); returns ln det(L + I) as a 0-d device tensor."""
    n, ld = Lc.shape[0], Lc.shape[1]
    cplx = Lc.dtype == torch.complex128
    op = DPP_OP_HERM_Z if cplx else DPP_OP_HERM_D
    logdet = torch.empty((), dtype=torch.float64, device=Lc.device)
    if work is None:
        work = torch.empty(max(dpp_lensemble_workspace_bytes(op, n), 256), dtype=torch.uint8, device=Lc.device)
    (dpp_lensemble_to_marginal_z if cplx else dpp_lensemble_to_marginal_d)(n, Lc, ld, logdet, work, stream=stream)
    return logdet


def dpp_philox_uniforms(seed, j0, b, count, u, stream=None):
    _check(_lib.dpp_philox_uniforms(seed, j0, b, count, _ptr(u), _stream(stream)))


def dpp_bcc_local_cols(n, nb, nranks, rank) -> int:
    return int(_lib.dpp_bcc_local_cols(n, nb, nranks, rank))


def dpp_dist_workspace_bytes(op, n, nranks, opts=None) -> int:
    return int(_lib.dpp_dist_workspace_bytes(op, n, nranks, _optp(opts)))


def dpp_comm_init(unique_id: bytes, nranks: int, rank: int):
    assert len(unique_id) == 128
    buf = ctypes.create_string_buffer(bytes(unique_id), 128)
    c = _P()
    _check(_lib.dpp_comm_init(buf, nranks, rank, ctypes.byref(c)))
    return c


def dpp_comm_init_local(nranks: int):
    c = _P()
    _check(_lib.dpp_comm_init_local(nranks, ctypes.byref(c)))
    return c


def dpp_dist_message_bytes(op, n, nranks, k) -> int:
    return int(_lib.dpp_dist_message_bytes(op, n, nranks, k))


def _ptr_array(ts):
    arr = (ctypes.c_void_p * len(ts))()
    for i, t in enumerate(ts):
        arr[i] = _ptr(t)
    return arr


def _dist_local(name):
    fn = getattr(_lib, name)

    def call(comm, n, K_locals, ld_local, seed, masks, loglik, info=None, opts=None, works=None, work_bytes=None,
             stream=None):
        """K_locals, masks, works: one device tensor per virtual rank; loglik (info): device arrays of
        nranks doubles (dpp_info_t)."""
        wb = work_bytes if work_bytes is not None else min(w.numel() for w in works)
        _check(fn(comm, n, _ptr_array(K_locals), ld_local, seed, _ptr_array(masks), _ptr(loglik), _ptr(info),
                  _optp(opts), _ptr_array(works), wb, _stream(stream)))
    call.__name__ = name
    return call


dpp_sample_herm_d_dist_local = _dist_local("dpp_sample_herm_d_dist_local")
dpp_sample_herm_z_dist_local = _dist_local("dpp_sample_herm_z_dist_local")


def dpp_comm_destroy(comm):
    _check(_lib.dpp_comm_destroy(comm))


def dpp_sample_herm_d_dist(comm, n, K_local, ld_local, seed, mask, loglik, info=None, opts=None, work=None,
                           work_bytes=None, stream=None):
    _check(_lib.dpp_sample_herm_d_dist(comm, n, _ptr(K_local), ld_local, seed, _ptr(mask), _ptr(loglik),
                                       _ptr(info), _optp(opts), _ptr(work),
                                       work_bytes if work_bytes is not None else work.numel(), _stream(stream)))


def dpp_sample_herm_z_dist(comm, n, K_local, ld_local, seed, mask, loglik, info=None, opts=None, work=None,
                           work_bytes=None, stream=None):
    _check(_lib.dpp_sample_herm_z_dist(comm, n, _ptr(K_local), ld_local, seed, _ptr(mask), _ptr(loglik),
                                       _ptr(info), _optp(opts), _ptr(work),
                                       work_bytes if work_bytes is not None else work.numel(), _stream(stream)))


STAGES = ("diag", "panel", "update_lookahead", "update_trailing", "aux")


def dpp_profile_begin():
    _check(_lib.dpp_profile_begin())


def dpp_profile_begin_stages(stage_mask: int):
    """Record only the stages whose bit (1 << STAGES.index(name)) is set."""
    _check(_lib.dpp_profile_begin_stages(stage_mask))


def dpp_profile_end() -> dict:
    p = dpp_profile_t()
    _check(_lib.dpp_profile_end(ctypes.byref(p)))
    return {st: dict(launches=int(p.launches[i]), ms=float(p.ms[i]), flops=float(p.flops[i]),
                     ms_union=float(p.ms_union[i]), top_flops=float(p.top_flops[i]), top_ms=float(p.top_ms[i]))
            for i, st in enumerate(STAGES)}


def dpp_profile_end_records(max_records: int = 1 << 16):
    """(per-stage aggregates as dpp_profile_end, timeline rows (stage name, start ms, end ms, flops))."""
    import numpy as np
    p = dpp_profile_t()
    buf = np.zeros(4 * max_records, dtype=np.float64)
    cnt = ctypes.c_int64(0)
    _check(_lib.dpp_profile_end_records(ctypes.byref(p), buf.ctypes.data, max_records, ctypes.byref(cnt)))
    agg = {st: dict(launches=int(p.launches[i]), ms=float(p.ms[i]), flops=float(p.flops[i]),
                    ms_union=float(p.ms_union[i]), top_flops=float(p.top_flops[i]), top_ms=float(p.top_ms[i]))
           for i, st in enumerate(STAGES)}
    n = min(int(cnt.value), max_records)
    rows = [(STAGES[int(buf[4 * i])], float(buf[4 * i + 1]), float(buf[4 * i + 2]), float(buf[4 * i + 3]))
            for i in range(n)]
    return agg, rows


def dpp_probe_update_d(m, K, W, L, ldo, C, ldc, stream=None) -> float:
    """One isolated launch of the real trailing-update kernel (C -= W L^T, lower triangle); its ms."""
    ms = ctypes.c_float(0.0)
    _check(_lib.dpp_probe_update_d(m, K, _ptr(W), _ptr(L), ldo, _ptr(C), ldc, ctypes.byref(ms), _stream(stream)))
    return float(ms.value)


def dpp_version() -> str:
    return _lib.dpp_version().decode()


# ------------------------------------------------------------------ conveniences
@dataclass
class Sample:
    mask: torch.Tensor     # uint8 [n] or [batch, n]
    loglik: torch.Tensor   # float64 [] or [batch]
    info: torch.Tensor     # uint8 [32] or [batch, 32] (dpp_info_t)

    def info_dicts(self):
        raw = self.info.reshape(-1, INFO_BYTES).cpu().numpy()
        out = []
        for row in raw:
            i = dpp_info_t.from_buffer_copy(row.tobytes())
            out.append(dict(n_kept=i.n_kept, n_ties=i.n_ties, first_tie=i.first_tie,
                            n_out_of_range=i.n_out_of_range, min_abs_pivot=i.min_abs_pivot,
                            max_abs_imag_pivot=i.max_abs_imag_pivot))
        return out


def colmajor(K: torch.Tensor) -> torch.Tensor:
    """Column-major storage (cols, ld=rows) of a naturally indexed matrix."""
    return K.transpose(0, 1).contiguous()


_OPS = {"herm_d": DPP_OP_HERM_D, "herm_z": DPP_OP_HERM_Z, "lu_z": DPP_OP_LU_Z, "herm_s": DPP_OP_HERM_S,
        "lu_c": DPP_OP_LU_C}
_INPLACE = {"herm_d": dpp_sample_herm_d, "herm_z": dpp_sample_herm_z, "lu_z": dpp_sample_lu_z,
            "herm_s": dpp_sample_herm_s, "lu_c": dpp_sample_lu_c}
_BATCHED = {"herm_d": dpp_sample_herm_d_batched, "herm_z": dpp_sample_herm_z_batched,
            "lu_z": dpp_sample_lu_z_batched, "herm_s": dpp_sample_herm_s_batched, "lu_c": dpp_sample_lu_c_batched}


def workspace(kind: str, n: int, batch: int = 1, batched: bool = False, opts=None, device="cuda"):
    op = _OPS[kind] | (DPP_OP_BATCHED if batched else 0)
    nbytes = dpp_workspace_bytes(op, batch, n, opts)
    return torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)


def sample(kind: str, Kc: torch.Tensor, seed: int = 0, opts=None, work=None, stream=None) -> Sample:
    """One sample (b = 0); Kc (column-major storage, shape (n, ld)) is OVERWRITTEN by the factor."""
    n, ld = Kc.shape[0], Kc.shape[1]
    dev = Kc.device
    mask = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
    ll = torch.empty((), dtype=torch.float64, device=dev)
    info = torch.empty(INFO_BYTES, dtype=torch.uint8, device=dev)
    if work is None:
        work = workspace(kind, n, opts=opts, device=dev)
    _INPLACE[kind](n, Kc, ld, seed, mask, ll, info, opts, work, stream=stream)
    return Sample(mask[:n], ll, info)


_MAP = {"herm_d": dpp_map_herm_d, "herm_z": dpp_map_herm_z, "lu_z": dpp_map_lu_z}


def greedy_map(kind: str, Kc: torch.Tensor, opts=None, work=None, stream=None) -> Sample:
    """Greedy MAP inference; Kc (column-major storage) is OVERWRITTEN."""
    n, ld = Kc.shape[0], Kc.shape[1]
    dev = Kc.device
    mask = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
    ll = torch.empty((), dtype=torch.float64, device=dev)
    info = torch.empty(INFO_BYTES, dtype=torch.uint8, device=dev)
    if work is None:
        work = workspace(kind, n, opts=opts, device=dev)
    _MAP[kind](n, Kc, ld, mask, ll, info, opts, work, stream=stream)
    return Sample(mask[:n], ll, info)


def sample_batched(kind: str, Kc: torch.Tensor, batch: int, seed: int = 0, b0: int = 0, strideK: int = 0,
                   opts=None, work=None, stream=None) -> Sample:
    """`batch` independent samples b0.. of the (read-only) kernel(s) in Kc."""
    if Kc.dim() == 3:
        n, ld = Kc.shape[1], Kc.shape[2]
        strideK = strideK or n * ld
    else:
        n, ld = Kc.shape[0], Kc.shape[1]
    dev = Kc.device
    mask = torch.empty((batch, max(n, 1)), dtype=torch.uint8, device=dev)
    ll = torch.empty(batch, dtype=torch.float64, device=dev)
    info = torch.empty((batch, INFO_BYTES), dtype=torch.uint8, device=dev)
    if work is None:
        work = workspace(kind, n, batch, batched=True, opts=opts, device=dev)
    _BATCHED[kind](batch, n, Kc, ld, strideK, seed, b0, mask, ll, info, opts, work, stream=stream)
    return Sample(mask[:, :n], ll, info)


def uniforms(seed: int, j0: int, b: int, count: int, device="cuda") -> torch.Tensor:
    u = torch.empty(max(count, 1), dtype=torch.float64, device=device)
    dpp_philox_uniforms(seed, j0, b, count, u)
    return u[:count]
