"""Seeded synthetic marginal kernels shaped like the paper's workloads.

This module holds NONE of the sampler's arithmetic (no pivot decisions, no
Schur updates, no Philox).  It only builds input kernels K and validates the
combinatorial structure of samples.  Both the CPU oracle (``oracle/``) and the
CUDA product path consume its outputs; neither is imported here.

Recipes:
  * ``haar_kernel``    K = Q diag(lam) Q^H, Q from QR of an i.i.d. Gaussian with
                       the Haar sign fix Q <- Q sign(diag R); lam ~ U(0,1) or
                       Beta(1/2,1/2); exactly symmetrised (BASELINE.json configs
                       0, 3, 4; Macchi's criterion PAPER.md:202-204 makes it
                       admissible).
  * ``ust_kernel``     transfer-current kernel K = B^T (B B^T)^{-1} B of a grid
                       graph with vertex 0 grounded (configs 1; PAPER.md:49-52,
                       81-83, 1159-1161).
  * ``aztec_kernel``   Kenyon's kernel M_ij = Kast(b_i,w_i) Kast^{-1}(w_i,b_j) of
                       the Aztec diamond (config 2).
  * ``similarity``     D^{-1} K D, a non-Hermitian kernel with the same DPP
                       (Prop. 2).
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "haar_kernel", "haar_kernel_torch", "projection_kernel", "ust_kernel", "grid_edges",
    "aztec_edges", "aztec_kernel", "similarity", "is_spanning_tree", "is_aztec_tiling",
    "log_num_spanning_trees_grid",
]


# --------------------------------------------------------------------------- Haar
def _haar_q(rng: np.random.Generator, n: int, complex_: bool) -> np.ndarray:
    if complex_:
        G = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(2.0)
    else:
        G = rng.standard_normal((n, n))
    Q, R = np.linalg.qr(G)
    d = np.diagonal(R)
    ph = d / np.abs(d)
    return Q * ph[None, :]


def _spectrum(rng: np.random.Generator, n: int, spectrum: str) -> np.ndarray:
    if spectrum == "uniform":
        return rng.uniform(0.0, 1.0, n)
    if spectrum == "beta":
        return rng.beta(0.5, 0.5, n)
    if spectrum.startswith("projection:"):
        r = int(spectrum.split(":")[1])
        lam = np.zeros(n)
        lam[:r] = 1.0
        return lam
    raise ValueError(spectrum)


def haar_kernel(n: int, seed: int = 0, spectrum: str = "uniform", complex_: bool = False) -> np.ndarray:
    """K = Q diag(lam) Q^H (numpy, host).  G is drawn first, then lam."""
    rng = np.random.default_rng(seed)
    Q = _haar_q(rng, n, complex_)
    lam = _spectrum(rng, n, spectrum)
    K = (Q * lam[None, :]) @ Q.conj().T
    K = 0.5 * (K + K.conj().T)
    if complex_:
        K[np.diag_indices(n)] = K.diagonal().real
    return np.asfortranarray(K)


def projection_kernel(n: int, rank: int, seed: int = 0, complex_: bool = False) -> np.ndarray:
    return haar_kernel(n, seed, f"projection:{rank}", complex_)


def haar_kernel_torch(n: int, seed: int = 0, spectrum: str = "uniform", complex_: bool = False,
                      device: str = "cuda"):
    """Same recipe on the GPU with torch (harness code for n >= 4096; untimed).

    Returns a torch tensor holding K in column-major order (i.e. a C-contiguous
    tensor T with T[l, i] = K[i, l]; K is symmetric/Hermitian so T = conj(K))."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    dt = torch.complex128 if complex_ else torch.float64
    if complex_:
        G = torch.complex(torch.randn(n, n, generator=g, device=device, dtype=torch.float64),
                          torch.randn(n, n, generator=g, device=device, dtype=torch.float64)) / np.sqrt(2.0)
    else:
        G = torch.randn(n, n, generator=g, device=device, dtype=torch.float64)
    Q, R = torch.linalg.qr(G)
    del G
    d = torch.diagonal(R)
    Q = Q * (d / d.abs())[None, :]
    del R
    if spectrum == "uniform":
        lam = torch.rand(n, generator=g, device=device, dtype=torch.float64)
    elif spectrum == "beta":
        # Beta(1/2, 1/2) by inverse CDF: x = sin^2(pi u / 2)
        u = torch.rand(n, generator=g, device=device, dtype=torch.float64)
        lam = torch.sin(0.5 * np.pi * u) ** 2
    else:
        raise ValueError(spectrum)
    K = (Q * lam.to(dt)[None, :]) @ Q.conj().T
    del Q
    K = 0.5 * (K + K.conj().T)
    if complex_:
        K.diagonal().imag.zero_()
    # column-major storage of K == row-major storage of K^T; for Hermitian K, K^T = conj(K)
    return K.T.contiguous()


def haar_kernel_bcc_torch(n: int, nb: int, world: int, rank: int, seed: int = 0, spectrum: str = "uniform",
                          complex_: bool = False, device: str = "cuda", chunk: int = 4096):
    """The same Haar recipe (G drawn first, then lam; Q from a Householder QR of G with the sign
    fix) for the 1D block-column-cyclic layout at large n (configs[4]: n = 65536 real, 34 GB per
    copy; n = 32768 complex): returns this rank's local storage L (ncols_local x n, C-contiguous)
    with L[q, i] = K(i, cols[q]), cols = the rank's global columns in block-cyclic order.  Memory:
    G and the QR factors are never alive together with K; K = (Q lam^1/2)(Q lam^1/2)^H is formed
    chunk by chunk.  Every rank draws the same G and lam (same seed), so the ranks' columns
    belong to one kernel."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    dt = torch.complex128 if complex_ else torch.float64
    if complex_:
        G = torch.complex(torch.randn(n, n, generator=g, device=device, dtype=torch.float64),
                          torch.randn(n, n, generator=g, device=device, dtype=torch.float64)) / np.sqrt(2.0)
    else:
        G = torch.randn(n, n, generator=g, device=device, dtype=torch.float64)
    a, tau = torch.geqrf(G)
    del G
    d = torch.diagonal(a).clone()
    Q = torch.linalg.householder_product(a, tau)
    del a, tau
    if spectrum == "uniform":
        lam = torch.rand(n, generator=g, device=device, dtype=torch.float64)
    elif spectrum == "beta":
        u = torch.rand(n, generator=g, device=device, dtype=torch.float64)
        lam = torch.sin(0.5 * np.pi * u) ** 2
    else:
        raise ValueError(spectrum)
    Q.mul_(((d / d.abs()) * lam.sqrt().to(dt))[None, :])   # Q <- Q phase(diag R) lam^1/2
    nblk = (n + nb - 1) // nb
    cols = [torch.arange(c * nb, min(n, (c + 1) * nb), device=device) for c in range(rank, nblk, world)]
    cols = torch.cat(cols) if cols else torch.zeros(0, dtype=torch.long, device=device)
    L = torch.empty((max(len(cols), 1), n), dtype=dt, device=device)
    for c0 in range(0, len(cols), chunk):
        rows = Q.index_select(0, cols[c0:c0 + chunk])          # Q(cols[q], :)
        L[c0:c0 + len(rows)] = (rows.conj() if complex_ else rows) @ Q.T
    del Q
    return L


# --------------------------------------------------------------------------- UST
def grid_edges(rows: int, cols: int):
    """Edges of a rows x cols grid graph; vertex id = y*cols + x.  Horizontal
    edges in row-major order, then vertical edges (reading #14)."""
    edges = []
    for y in range(rows):
        for x in range(cols - 1):
            edges.append((y * cols + x, y * cols + x + 1))
    for y in range(rows - 1):
        for x in range(cols):
            edges.append((y * cols + x, (y + 1) * cols + x))
    return edges


def ust_kernel(rows: int, cols: int) -> np.ndarray:
    """Transfer-current kernel K = B^T (B B^T)^{-1} B, B = reduced incidence
    matrix (vertex 0 grounded); +1 at the lower vertex id, -1 at the higher."""
    import scipy.linalg as sla
    edges = grid_edges(rows, cols)
    V, E = rows * cols, len(edges)
    B = np.zeros((V, E))
    for e, (a, b) in enumerate(edges):
        B[a, e] = 1.0
        B[b, e] = -1.0
    B = B[1:, :]
    L = B @ B.T
    c = sla.cho_factor(L, lower=True)
    X = sla.cho_solve(c, B)
    K = B.T @ X
    K = 0.5 * (K + K.T)
    return np.asfortranarray(K)


def is_spanning_tree(V: int, edges, kept: np.ndarray) -> bool:
    sel = [edges[e] for e in np.flatnonzero(kept)]
    if len(sel) != V - 1:
        return False
    parent = list(range(V))

    def find(a):
        while parent[a] != a:
            parent[a] = parent[parent[a]]
            a = parent[a]
        return a

    for a, b in sel:
        ra, rb = find(a), find(b)
        if ra == rb:
            return False
        parent[ra] = rb
    return True


def log_num_spanning_trees_grid(rows: int, cols: int) -> float:
    """ln tau(P_rows x P_cols) from the Laplacian eigenvalue product (Kirchhoff):
    tau = (1/V) prod_{(j,k) != (0,0)} (4 - 2cos(pi j/rows) - 2cos(pi k/cols))."""
    s = 0.0
    for j in range(rows):
        for k in range(cols):
            if j == 0 and k == 0:
                continue
            s += np.log(4.0 - 2.0 * np.cos(np.pi * j / rows) - 2.0 * np.cos(np.pi * k / cols))
    return s - np.log(rows * cols)


# --------------------------------------------------------------------------- Aztec
def aztec_squares(d: int):
    """Unit squares (lower-left corner (x, y)) of the order-d Aztec diamond."""
    sq = []
    for x in range(-d, d):
        for y in range(-d, d):
            if abs(x + 0.5) + abs(y + 0.5) <= d:
                sq.append((x, y))
    return sq


def aztec_edges(d: int):
    """Ground set: adjacent (black, white) square pairs; black iff x+y even.
    Black squares sorted by (x, y); neighbours in order E, W, N, S (reading #15).
    Returns (edges, blacks, whites) with edges = [(bi, wi, vertical: bool)]."""
    sq = aztec_squares(d)
    sset = set(sq)
    blacks = sorted([s for s in sq if (s[0] + s[1]) % 2 == 0])
    whites = sorted([s for s in sq if (s[0] + s[1]) % 2 != 0])
    widx = {w: i for i, w in enumerate(whites)}
    edges = []
    for bi, (x, y) in enumerate(blacks):
        for dx, dy, vert in ((1, 0, False), (-1, 0, False), (0, 1, True), (0, -1, True)):
            nb = (x + dx, y + dy)
            if nb in sset:
                edges.append((bi, widx[nb], vert))
    return edges, blacks, whites


def aztec_kernel(d: int) -> np.ndarray:
    """Kenyon's kernel M_ij = Kast(b_i, w_i) Kast^{-1}(w_i, b_j) (plain gauge).

    The plain gauge is fine in fp64 up to d ~ 20;
    larger d needs the balanced gauge (not built in round 1)."""
    edges, blacks, whites = aztec_edges(d)
    nb = len(blacks)
    Kast = np.zeros((nb, len(whites)), dtype=np.complex128)
    for bi, wi, vert in edges:
        Kast[bi, wi] = 1j if vert else 1.0
    Kinv = np.linalg.inv(Kast)
    n = len(edges)
    bidx = np.array([e[0] for e in edges])
    widx = np.array([e[1] for e in edges])
    kv = np.array([1j if e[2] else 1.0 for e in edges])
    M = kv[:, None] * Kinv[widx][:, bidx]
    assert M.shape == (n, n)
    return np.asfortranarray(M)


def _aztec_kast_torch(d: int, a_exp: dict, c_exp: dict, device: str):
    """Gauged Kasteleyn matrix K'(b, w) = 2^{a_b} Kast(b, w) 2^{c_w} (exact: powers of two) and the
    edge list; a_exp / c_exp map square -> integer exponent (missing squares: 0)."""
    import torch
    edges, blacks, whites = aztec_edges(d)
    m = len(blacks)
    a = torch.tensor([float(a_exp.get(s, 0)) for s in blacks], dtype=torch.float64)
    c = torch.tensor([float(c_exp.get(s, 0)) for s in whites], dtype=torch.float64)
    K = torch.zeros((m, m), dtype=torch.complex128)
    bi = torch.tensor([e[0] for e in edges])
    wi = torch.tensor([e[1] for e in edges])
    kv = torch.tensor([1j if e[2] else 1.0 for e in edges], dtype=torch.complex128)
    K[bi, wi] = kv * torch.exp2(a[bi] + c[wi]).to(torch.complex128)
    return K.to(device), a.to(device), c.to(device), edges, blacks, whites


def _osborne_bipartite(Kp, Ki, a, c, rounds: int = 40):
    """Osborne balancing of Z = [[0, K'], [K'^{-1}, 0]] with power-of-two scalings, sweeping all
    black indices, then all white ones (Z is bipartite, so a simultaneous sweep over one colour IS
    the sequential Osborne sweep).  Scales Kp, Ki in place (exactly) and updates the exponents."""
    import torch
    for _ in range(rounds):
        changed = False
        # black b: row b of Z = K'(b, :), column b of Z = K'^{-1}(:, b)
        r = Kp.abs().sum(dim=1)
        cc = Ki.abs().sum(dim=0)
        e = torch.round(0.5 * torch.log2(r / cc))
        if bool((e != 0).any()):
            changed = True
            a -= e
            Kp *= torch.exp2(-e).to(Kp.dtype)[:, None]
            Ki *= torch.exp2(e).to(Ki.dtype)[None, :]
        # white w: row w of Z = K'^{-1}(w, :), column w of Z = K'(:, w)
        r = Ki.abs().sum(dim=1)
        cc = Kp.abs().sum(dim=0)
        e = torch.round(0.5 * torch.log2(r / cc))
        if bool((e != 0).any()):
            changed = True
            c += e
            Ki *= torch.exp2(-e).to(Ki.dtype)[:, None]
            Kp *= torch.exp2(e).to(Kp.dtype)[None, :]
        if not changed:
            break


def aztec_kernel_balanced(d: int, device: str = "cpu", d_start: int = 20, d_step: int = 5,
                          passes: int = 2, storage: str = "colmajor", return_info: bool = False):
    """Kenyon's kernel of the order-d Aztec diamond in an Osborne-balanced gauge (reading R13;
    SURVEY.md Appendix A.5), built with torch on `device` (harness code, not the method).

    M'_ij = K'(b_i, w_i) K'^{-1}(w_i, b_j) with K' = diag(2^a) Kast diag(2^c).  Then
    M' = D M D^{-1} with D_ii = 2^{a(b_i)}, which defines the same DPP as Kenyon's M (Prop. 2,
    PAPER.md:178-195) but stays well conditioned in fp64 at d = 80, where the plain gauge's
    inverse is garbage (max|Kast^{-1}| ~ 7e21).  Exponents are found at d_start (plain gauge,
    accurate there) and carried outward in steps of d_step: each new square takes the exponent of
    the nearest same-colour square inward along the diagonal, then `passes` rounds of
    (invert, balance) fix them up.

    storage="colmajor" returns a torch tensor T (n x n, C-contiguous) with T[j, i] = M'[i, j]
    (the sampler's column-major layout); "natural" returns M' itself."""
    import torch
    a_exp: dict = {}
    c_exp: dict = {}
    dd = min(d, d_start)
    info = {"steps": []}
    while True:
        Kp, a, c, edges, blacks, whites = _aztec_kast_torch(dd, a_exp, c_exp, device)
        for _ in range(passes):
            Ki = torch.linalg.inv(Kp)
            _osborne_bipartite(Kp, Ki, a, c)
        Ki = torch.linalg.inv(Kp)
        eye = torch.eye(Kp.shape[0], dtype=Kp.dtype, device=Kp.device)
        res = float((Kp @ Ki - eye).abs().max())
        info["steps"].append({"d": dd, "inverse_residual": res, "max_abs_Kinv": float(Ki.abs().max())})
        a_exp = {s: int(v) for s, v in zip(blacks, a.cpu().tolist())}
        c_exp = {s: int(v) for s, v in zip(whites, c.cpu().tolist())}
        if dd == d:
            break
        dn = min(d, dd + d_step)
        # seed the new squares from the nearest same-colour square inward along the diagonal
        for x, y in aztec_squares(dn):
            s = (x, y)
            tgt = a_exp if (x + y) % 2 == 0 else c_exp
            if s in tgt:
                continue
            px, py = x, y
            while (px, py) not in tgt:  # each diagonal step lowers |x+1/2| + |y+1/2| by >= 1
                px, py = px - (1 if px + 0.5 > 0 else -1), py - (1 if py + 0.5 > 0 else -1)
            tgt[s] = tgt[(px, py)]
        dd = dn
    bidx = torch.tensor([e[0] for e in edges], device=Kp.device)
    widx = torch.tensor([e[1] for e in edges], device=Kp.device)
    kd = Kp[bidx, widx]                                   # K'(b_i, w_i)
    if storage == "colmajor":
        # T[j, i] = M'[i, j] = kd_i Ki[w_i, b_j] = kd_i (Ki^T)[b_j, w_i]
        T = Ki.T.contiguous()[bidx]                       # n x m: rows b_j
        T = T[:, widx] * kd[None, :]
    else:
        T = kd[:, None] * Ki[widx][:, bidx]
    if return_info:
        info["a_black"] = a.cpu().numpy()
        info["edges"] = edges
        return T, info
    return T


def is_aztec_tiling(d: int, kept: np.ndarray) -> bool:
    edges, blacks, whites = aztec_edges(d)
    sel = np.flatnonzero(kept)
    if len(sel) != d * (d + 1):
        return False
    bc = np.zeros(len(blacks), dtype=int)
    wc = np.zeros(len(whites), dtype=int)
    for e in sel:
        bc[edges[e][0]] += 1
        wc[edges[e][1]] += 1
    return bool(np.all(bc == 1) and np.all(wc == 1))


# --------------------------------------------------------------------------- Prop. 2
def similarity(K: np.ndarray, seed: int = 0, lo: float = 0.5, hi: float = 2.0) -> np.ndarray:
    """D^{-1} K D with a random complex diagonal D, |D| in [lo, hi] (Prop. 2)."""
    rng = np.random.default_rng(seed + 7919)
    n = K.shape[0]
    mag = rng.uniform(lo, hi, n)
    ph = np.exp(2j * np.pi * rng.uniform(0, 1, n))
    D = mag * ph
    return np.asfortranarray((1.0 / D)[:, None] * K.astype(np.complex128) * D[None, :])
