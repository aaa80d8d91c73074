"""Multi-GPU plumbing for the two partitioned modes; no arithmetic of the method.

* Independent samples: ``shard_samples`` splits the sample indices b across ranks (each rank
  calls the batched C entry point with its own b0); no data-path collective.
* 1D block-column-cyclic factorization: rank r of P owns block columns c = r, r+P, ... of width
  nb.  ``bcc_columns`` lists the global columns a rank owns (in local storage order),
  ``to_local`` / ``from_local`` move between a full matrix and a rank's local storage, and
  ``DistComm`` wraps the library's NCCL communicator (``dpp_comm_init``), created from a unique id
  that rank 0 draws and ``torch.distributed.broadcast_object_list`` distributes.
The sampling itself (diag / panel / broadcast / update) runs inside ``dpp_sample_herm_{d,z}_dist``.
"""
from __future__ import annotations

import numpy as np
import torch


def shard_samples(batch: int, world: int, rank: int):
    """Contiguous shard (b0, count) of `batch` sample indices for `rank`."""
    per, extra = divmod(batch, world)
    b0 = rank * per + min(rank, extra)
    return b0, per + (1 if rank < extra else 0)


def bcc_columns(n: int, nb: int, world: int, rank: int) -> np.ndarray:
    """Global column indices owned by `rank`, in local storage order."""
    nblk = (n + nb - 1) // nb
    cols = [np.arange(c * nb, min(n, (c + 1) * nb)) for c in range(rank, nblk, world)]
    return np.concatenate(cols) if cols else np.zeros(0, dtype=np.int64)


def owner_of_block(k: int, world: int) -> int:
    return k % world


def to_local(K_colmajor: torch.Tensor, n: int, nb: int, world: int, rank: int, ld_local: int | None = None):
    """Local storage (ncols_local, ld_local) of a rank, from the full column-major storage
    (cols, ld) of K: local column q holds global column bcc_columns(...)[q]."""
    cols = torch.as_tensor(bcc_columns(n, nb, world, rank), device=K_colmajor.device)
    ld_local = ld_local or max(n, 1)
    out = torch.zeros((max(len(cols), 1), ld_local), dtype=K_colmajor.dtype, device=K_colmajor.device)
    if len(cols):
        out[: len(cols), :n] = K_colmajor.index_select(0, cols)[:, :n]
    return out


def from_local(locals_: list, n: int, nb: int, world: int, like: torch.Tensor) -> torch.Tensor:
    """Reassemble the full column-major storage from every rank's local storage."""
    full = torch.zeros((n, n), dtype=like.dtype, device=like.device)
    for r, loc in enumerate(locals_):
        cols = torch.as_tensor(bcc_columns(n, nb, world, r), device=like.device)
        if len(cols):
            full.index_copy_(0, cols, loc[: len(cols), :n].to(like.device))
    return full


def message_bytes(n: int, nb: int, k: int, elem_bytes: int = 8) -> int:
    """Bytes broadcast at block step k with P > 1 (mirrors csrc/dist.cu and
    dpp_dist_message_bytes: a 256-byte-aligned header [state 64 B | D1 | decisions] + L21 of the
    LIVE rows m2 = n - j1 at pitch round_up(m2, 16); elem_bytes 8 real, 16 complex Hermitian)."""
    header = 64 + 8 * nb + nb
    header = (header + 255) // 256 * 256
    j1 = min(n, (k + 1) * nb)
    jb = min(nb, n - k * nb)
    m2 = n - j1
    pitch = max(((m2 + 15) // 16) * 16, 16)
    return header + (pitch * jb * elem_bytes if m2 > 0 else 0)


def sample_local(locals_: list, n: int, seed: int, complex_: bool = False, opts=None, stream=None):
    """One sample with the block columns spread over len(locals_) VIRTUAL ranks on the current
    device (dpp_comm_init_local + dpp_sample_herm_{d,z}_dist_local): locals_[r] is rank r's local
    storage (ncols_local, ld_local).  Returns {"masks": [P x n uint8], "loglik": [P], "info": [P x 32
    bytes]} -- every virtual rank's copy of the result."""
    from . import (DPP_OP_HERM_D, DPP_OP_HERM_Z, INFO_BYTES, dpp_comm_destroy, dpp_comm_init_local,
                   dpp_dist_workspace_bytes, dpp_sample_herm_d_dist_local, dpp_sample_herm_z_dist_local)
    P = len(locals_)
    dev = locals_[0].device
    op = DPP_OP_HERM_Z if complex_ else DPP_OP_HERM_D
    wb = dpp_dist_workspace_bytes(op, n, P, opts)
    works = [torch.empty(max(wb, 256), dtype=torch.uint8, device=dev) for _ in range(P)]
    masks = torch.empty((P, max(n, 1)), dtype=torch.uint8, device=dev)
    ll = torch.empty(P, dtype=torch.float64, device=dev)
    info = torch.empty((P, INFO_BYTES), dtype=torch.uint8, device=dev)
    comm = dpp_comm_init_local(P)
    try:
        fn = dpp_sample_herm_z_dist_local if complex_ else dpp_sample_herm_d_dist_local
        fn(comm, n, locals_, locals_[0].shape[1], seed, [masks[r] for r in range(P)], ll, info, opts, works,
           work_bytes=wb, stream=stream)
        torch.cuda.synchronize(dev)
    finally:
        dpp_comm_destroy(comm)
    return {"masks": masks[:, :n], "loglik": ll, "info": info}


class DistComm:
    """The library's NCCL communicator for the block-cyclic mode, bootstrapped over an existing
    torch.distributed process group (any backend) by sharing rank 0's NCCL unique id."""

    def __init__(self, group=None):
        import torch.distributed as dist
        from . import dpp_comm_init
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        uid = [unique_id() if self.rank == 0 else None]
        dist.broadcast_object_list(uid, src=0, group=group)
        self.unique_id = uid[0]
        self.handle = dpp_comm_init(self.unique_id, self.world, self.rank)

    def close(self):
        from . import dpp_comm_destroy
        if self.handle is not None:
            dpp_comm_destroy(self.handle)
            self.handle = None


def unique_id() -> bytes:
    """A fresh 128-byte ncclUniqueId (torch's bundled NCCL)."""
    return bytes(torch.cuda.nccl.unique_id())
