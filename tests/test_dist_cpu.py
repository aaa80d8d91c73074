"""World-size-2 gloo tests (CPU) of the multi-GPU host logic.

* independent-sample sharding covers every sample index exactly once;
* the block-column-cyclic layout of paper_1905_00165_b200.dist agrees with the C ABI
  (dpp_bcc_local_cols) and partitions the columns; to_local/from_local round-trip;
* the NCCL unique id travels over broadcast_object_list (the DistComm bootstrap);
* a numpy emulation of the distributed schedule of csrc/dist.cu -- owner factors tile + panel,
  broadcasts [D1 | decisions | running loglik | L21] (here over gloo), every rank updates its own
  trailing block columns, in the lookahead order of csrc/dist.cu -- reproduces the oracle's sample
  and factor for real and complex Hermitian kernels.  (The CUDA kernels of that
  schedule are covered on the GPU by tests/test_gpu_dist.py: world size 1 over NCCL and P = 2, 3, 4
  virtual ranks with the in-process transport, which runs the same per-step code.)
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _emulate(K, n, nb, world, rank, seed, oracle_mod):
    """Distributed blocked LDL^H DPP sampling with numpy compute and gloo broadcasts, in the
    lookahead order of csrc/dist.cu: with message k in hand, owner(k+1) updates block column k+1
    with it, factors tile + panel k+1 and broadcasts message k+1; only then does every rank apply
    step k to the rest of its trailing block columns.  Real or complex Hermitian K."""
    from paper_1905_00165_b200 import dist as D
    cplx = np.iscomplexobj(K)
    cols = D.bcc_columns(n, nb, world, rank)
    Kc = torch.from_numpy(np.ascontiguousarray(K.T))            # column-major storage
    loc = D.to_local(Kc, n, nb, world, rank).numpy().T.copy()  # natural: loc[:, q] = K[:, cols[q]]
    mask = np.zeros(n, dtype=np.uint8)
    ll = [0.0]
    nblk = (n + nb - 1) // nb
    msgs = {}

    def pitch(m2):  # the message's L21 pitch: the live rows, 16-aligned (csrc/dist.cu msg_pitch)
        return max(((m2 + 15) // 16) * 16, 16)

    def span(k):
        j0, j1 = k * nb, min(n, (k + 1) * nb)
        return j0, j1, j1 - j0, n - j1

    def factor(k):  # owner(k): stage 1 (Listing 1 on the tile, lower triangle) + stage 2, packed
        j0, j1, jb, m2 = span(k)
        q = np.searchsorted(cols, j0)
        T = loc[j0:j1, q:q + jb]
        for t in range(jb):
            d = T[t, t].real
            keep = oracle_mod.uniform(seed, j0 + t, 0) <= d
            if not keep:
                d -= 1.0
            T[t, t] = d
            mask[j0 + t] = keep
            ll[0] += np.log(abs(d))
            w = T[t + 1:, t].copy()
            T[t + 1:, t] = w / d
            T[t + 1:, t + 1:] -= np.tril(np.outer(T[t + 1:, t], w.conj()))
        Dg = np.diag(T).real.copy()
        L11 = np.tril(T, -1) + np.eye(jb)
        A21 = loc[j1:, q:q + jb]
        W21 = np.linalg.solve(L11, A21.conj().T).conj().T if m2 else np.zeros((0, jb))  # A21 L11^{-H}
        loc[j1:, q:q + jb] = W21 / Dg[None, :]                                         # L21
        buf = np.zeros((pitch(m2), jb), dtype=loc.dtype)
        buf[:m2] = loc[j1:, q:q + jb]
        return [ll[0], Dg, mask[j0:j1].copy(), buf]

    def exchange(k):  # ncclBroadcast(message k, root = owner(k)) -- here over gloo
        j0, j1, jb, m2 = span(k)
        owner = D.owner_of_block(k, world)
        ldw = pitch(m2)
        msg = torch.zeros(2 + 2 * jb + (2 if cplx else 1) * ldw * jb, dtype=torch.float64)
        if rank == owner:
            lk, Dg, mk, buf = msgs[k]
            msg[0] = lk
            msg[2:2 + jb] = torch.from_numpy(Dg)
            msg[2 + jb:2 + 2 * jb] = torch.from_numpy(mk.astype(np.float64))
            body = buf.T.reshape(-1)
            msg[2 + 2 * jb:] = torch.from_numpy(body.view(np.float64))
        dist.broadcast(msg, src=owner)
        ll[0] = float(msg[0])
        mask[j0:j1] = msg[2 + jb:2 + 2 * jb].numpy().astype(np.uint8)
        L21 = msg[2 + 2 * jb:].numpy().copy().view(loc.dtype).reshape(jb, ldw).T[:m2]
        msgs[k] = (msg[2:2 + jb].numpy().copy(), L21)

    def update(k, blocks):  # stage 3 of step k on the given local block columns: C -= L21 D1 L21^H
        j0, j1, jb, m2 = span(k)
        Dg, L21 = msgs[k]
        for qi, c in enumerate(cols):
            if c // nb in blocks:
                rows = np.arange(c, n)
                loc[rows, qi] -= L21[rows - j1] @ (L21[c - j1].conj() * Dg)

    if rank == D.owner_of_block(0, world):
        msgs[0] = factor(0)
    exchange(0)
    for k in range(nblk):
        if n - span(k)[1] == 0:
            break
        kn = k + 1
        if rank == D.owner_of_block(kn, world):
            update(k, {kn})           # lookahead: block column k+1 first
            msgs[kn] = factor(kn)
        exchange(kn)
        rest = {c // nb for c in cols if c // nb > kn or (c // nb == kn and rank != D.owner_of_block(kn, world))}
        update(k, rest)
    return loc, cols, mask, ll[0]


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import paper_1905_00165_b200 as dpp
        import workloads as W
        from paper_1905_00165_b200 import dist as D
        out = {}
        # (1) sample sharding
        b0, cnt = D.shard_samples(1001, world, rank)
        got = [None] * world
        dist.all_gather_object(got, list(range(b0, b0 + cnt)))
        out["shard_ok"] = sorted(sum(got, [])) == list(range(1001))
        # (2) block-cyclic layout vs the C ABI
        ok = True
        for n, nb in [(1000, 128), (16384, 128), (65536, 128), (130, 32), (5, 128)]:
            cols = D.bcc_columns(n, nb, world, rank)
            ok &= len(cols) == dpp.dpp_bcc_local_cols(n, nb, world, rank)
            allc = [None] * world
            dist.all_gather_object(allc, cols.tolist())
            ok &= sorted(sum(allc, [])) == list(range(n))
        out["layout_ok"] = ok
        # (3) unique-id bootstrap over the process group
        uid = [os.urandom(128) if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ids = [None] * world
        dist.all_gather_object(ids, uid[0])
        out["uid_ok"] = len(uid[0]) == 128 and ids[0] == ids[1]
        # (4) emulated distributed sampler (lookahead order) vs the oracle, real and complex
        n, nb, seed = 300, 32, 17
        for cplx in (False, True):
            K = W.haar_kernel(n, seed=3, complex_=cplx)
            loc, cols, mask, ll = _emulate(K.copy(), n, nb, world, rank, seed, oracle)
            pieces = [None] * world
            dist.all_gather_object(pieces, (cols.tolist(), loc[:, :len(cols)]))
            F = np.zeros((n, n), dtype=K.dtype)
            for cl, lc in pieces:
                F[:, cl] = lc
            o = (oracle.sample_herm_z if cplx else oracle.sample_herm_d)(K, seed, 0)
            tag = "z" if cplx else "d"
            out["mask_ok_" + tag] = bool(np.array_equal(mask, o.mask)) and o.n_ties == 0
            out["factor_err_" + tag] = float(np.max(np.abs(np.tril(F) - np.tril(o.factor))))
            out["ll_err_" + tag] = abs(ll - o.loglik) / abs(o.loglik)
        # round trip of the local storage helpers
        Kc = torch.from_numpy(np.ascontiguousarray(K.T))
        locs = [None] * world
        dist.all_gather_object(locs, D.to_local(Kc, n, nb, world, rank))
        out["roundtrip_ok"] = bool(torch.equal(D.from_local(locs, n, nb, world, Kc), Kc))
        out["msg0"] = D.message_bytes(16384, 128, 0)
        out["msg0z"] = D.message_bytes(32768, 64, 0, elem_bytes=16)
        # the Python mirror equals the library's dpp_dist_message_bytes at every step
        out["msg_mirror_ok"] = all(
            D.message_bytes(n_, nb_, k, es) == dpp.dpp_dist_message_bytes(op, n_, 2, k)
            for n_, nb_, es, op in ((1000, 128, 8, dpp.DPP_OP_HERM_D), (65536, 128, 8, dpp.DPP_OP_HERM_D),
                                    (777, 64, 16, dpp.DPP_OP_HERM_Z))
            for k in range((n_ + nb_ - 1) // nb_))
        # per receiver over a whole n = 65536 sample: ~ 4 n^2 bytes (the live rows only)
        out["msg_total_65536"] = sum(D.message_bytes(65536, 128, k) for k in range(512))
        results[rank] = out
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_host_logic():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, port, results), nprocs=world, join=True)
    for r in range(world):
        res = results[r]
        assert res["shard_ok"] and res["layout_ok"] and res["uid_ok"] and res["roundtrip_ok"], res
        for tag in ("d", "z"):
            assert res["mask_ok_" + tag], res
            assert res["factor_err_" + tag] < 1e-10, res
            assert res["ll_err_" + tag] < 1e-12, res
        # header (64 B state + 128 pivots + 128 decision bytes, 256-aligned) + L21 of the live rows
        # (m2 = n - nb, pitch round_up(m2, 16))
        assert res["msg0"] == 1280 + 16256 * 128 * 8, res
        assert res["msg0z"] == 768 + 32704 * 64 * 16, res
        assert res["msg_mirror_ok"], res
        assert abs(res["msg_total_65536"] / (4 * 65536 ** 2) - 1) < 0.01, res
