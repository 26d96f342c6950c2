"""CPU tests of the slab partition with world_size-2 gloo.

The device engine's multi-rank path (csrc/comm.cu) is: slabs along the
slowest axis, a ring halo exchange before every stencil consumer (my first
planes -> rank-1's high ghost, my last planes -> rank+1's low ghost), and an
all-reduce of every inner product.  Here the same decomposition is restated
on the CPU with the oracle's CSR operators and checked for P-independence:
slab-local stencil application with exchanged ghosts equals the global
operator, and a restarted CGS2 GMRES whose dot products are all-reduced takes
the same iterations and reaches the same solution as the single-domain
oracle (src/sparsela.py:176-280).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import irk
from oracle.problems import build_problem
from paper_2101_01776_b200.distributed import gather, pencil_layout, scatter, slab_range


def test_slab_ranges_tile_the_axis():
    for planes in (7, 24, 64, 4096):
        for p in (1, 2, 3, 8):
            if planes < p:
                continue
            ranges = [slab_range(planes, r, p) for r in range(p)]
            assert ranges[0][0] == 0
            assert all(a[0] + a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            assert sum(nl for _, nl in ranges) == planes
            assert max(nl for _, nl in ranges) - min(nl for _, nl in ranges) <= 1


@pytest.mark.parametrize("shape,p", [((8, 12), 2), ((5, 4, 9), 3), ((16, 16), 4)])
def test_scatter_gather_round_trip(shape, p):
    v = np.arange(int(np.prod(shape)), dtype=float)
    parts = [scatter(v, shape, r, p) for r in range(p)]
    assert np.array_equal(gather(parts, shape), v)


# ------------------------------------------------ 2-process gloo restatement


def _ring_halo(send_lo, send_hi, rank, nranks):
    """The engine's halo semantics (comm.cu) on CPU tensors."""
    prev, nxt = (rank - 1) % nranks, (rank + 1) % nranks
    r_hi = torch.empty_like(send_lo)
    r_lo = torch.empty_like(send_hi)
    reqs = [dist.isend(send_lo, prev, tag=0), dist.isend(send_hi, nxt, tag=1),
            dist.irecv(r_hi, nxt, tag=0), dist.irecv(r_lo, prev, tag=1)]
    for r in reqs:
        r.wait()
    return r_lo, r_hi


class SlabOperator:
    """Rows of a global stencil CSR owned by one slab, acting on the slab
    extended by one ghost plane on each side."""

    def __init__(self, A, shape, rank, nranks):
        planes, plane = shape[-1], int(np.prod(shape[:-1]))
        p0, nl = slab_range(planes, rank, nranks)
        self.plane, self.nl, self.rank, self.nranks = plane, nl, rank, nranks
        ext_planes = [(p0 - 1) % planes] + list(range(p0, p0 + nl)) + [(p0 + nl) % planes]
        cols = np.concatenate([np.arange(q * plane, (q + 1) * plane) for q in ext_planes])
        rows = np.arange(p0 * plane, (p0 + nl) * plane)
        self.A = A.tocsr()[rows][:, cols]
        assert abs(A.tocsr()[rows].sum() - self.A.sum()) < 1e-9 * (1 + abs(self.A.sum()))

    def __call__(self, x):
        lo, hi = _ring_halo(torch.from_numpy(x[: self.plane].copy()),
                            torch.from_numpy(x[-self.plane:].copy()), self.rank, self.nranks)
        return self.A @ np.concatenate([lo.numpy(), x, hi.numpy()])


def _allreduce(v):
    t = torch.from_numpy(np.atleast_1d(np.asarray(v, dtype=float)).copy())
    dist.all_reduce(t)
    return t.numpy()


def dist_gmres(apply_op, rhs, rtol, maxit, restart):
    """Restarted CGS2 GMRES (the reference control flow, src/sparsela.py:176-280)
    with every dot product all-reduced over the slabs."""
    dot = lambda a, b: float(_allreduce(a @ b)[0])  # noqa: E731
    n = rhs.size
    bnorm = np.sqrt(dot(rhs, rhs))
    x = np.zeros(n)
    r = rhs.copy()
    beta = bnorm
    total, converged = 0, False
    while not converged and total < maxit:
        m = min(restart, maxit - total)
        v = np.zeros((n, m + 1))
        h = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        v[:, 0] = r / beta
        g[0] = beta
        j = -1
        for j in range(m):
            w = apply_op(v[:, j])
            for _ in range(2):
                coef = _allreduce(v[:, : j + 1].T @ w)
                w -= v[:, : j + 1] @ coef
                h[: j + 1, j] += coef
            hj = np.sqrt(dot(w, w))
            h[j + 1, j] = hj
            v[:, j + 1] = w / hj
            for i in range(j):
                tmp = cs[i] * h[i, j] + sn[i] * h[i + 1, j]
                h[i + 1, j] = -sn[i] * h[i, j] + cs[i] * h[i + 1, j]
                h[i, j] = tmp
            denom = np.hypot(h[j, j], h[j + 1, j])
            cs[j], sn[j] = h[j, j] / denom, h[j + 1, j] / denom
            h[j, j], h[j + 1, j] = denom, 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            total += 1
            if abs(g[j + 1]) / bnorm <= rtol or total >= maxit:
                break
        k = j + 1
        y = np.zeros(k)
        for i in range(k - 1, -1, -1):
            y[i] = (g[i] - h[i, i + 1: k] @ y[i + 1: k]) / h[i, i]
        x = x + v[:, :k] @ y
        r = rhs - apply_op(x)
        beta = np.sqrt(dot(r, r))
        converged = beta / bnorm <= rtol
    return x, total, converged


def _worker(rank, nranks, port, kind, shape, queue):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=nranks)
    try:
        params = {"burgers": dict(nu=0.02), "nldiff": {}}[kind]
        pd = build_problem(kind, shape, **params)
        rng = np.random.default_rng(4)
        u = rng.standard_normal(pd.dim) * 0.3
        A_lin = pd.linearize_csr(u, 0.0)
        dt = 2e-3
        S = (3.0 * np.eye(pd.dim) - dt * A_lin.toarray())  # a shifted stage operator
        import scipy.sparse as sp

        S = sp.csr_matrix(S)
        op = SlabOperator(S, shape, rank, nranks)
        # 1) slab stencil == global operator rows
        x = rng.standard_normal(pd.dim)
        y_loc = op(scatter(x, shape, rank, nranks).copy())
        ok_apply = np.allclose(y_loc, scatter(S @ x, shape, rank, nranks), atol=1e-12)
        # 2) distributed GMRES == single-domain oracle GMRES
        b = rng.standard_normal(pd.dim)
        xl, its, conv = dist_gmres(op, scatter(b, shape, rank, nranks).copy(), 1e-10, 300, 15)
        xo, rep = irk.gmres(lambda z: S @ z, b, pd.dim, None, 0, 1e-10, 300, 15)
        parts = [None] * nranks
        dist.all_gather_object(parts, xl)
        if rank == 0:
            xg = gather(parts, shape)
            queue.put((bool(ok_apply), its, rep.iterations, bool(conv), rep.converged,
                       float(np.linalg.norm(xg - xo) / np.linalg.norm(xo))))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("kind,shape", [("burgers", (12, 10)), ("nldiff", (6, 5, 8))])
def test_two_rank_gloo_decomposition_is_p_independent(kind, shape):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, shape, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    ok_apply, its, its_ref, conv, conv_ref, rel = res
    assert ok_apply
    assert conv and conv_ref
    assert abs(its - its_ref) <= 1, (its, its_ref)
    assert rel <= 1e-8, rel


def _dae_worker(rank, nranks, port, shape, queue):
    """The multi-rank DAE path (csrc/dae.cu) restated: the Arakawa 9-point
    differential operator on slabs with one full ghost plane each side (the
    corners come with the planes), and the constraint solve on the gathered
    right-hand side -- each rank's slab zero-padded into the global vector and
    all-reduced (exact), solved globally, own slab kept.  (The device path
    replaced the gather by the slab -> pencil transpose FFT restated in
    _pencil_worker below; the gathered form stays as the P-independence check
    of the slab operators and of the pinned row.)"""
    import scipy.sparse.linalg as spla

    from oracle.problems import DaeProblemDef

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=nranks)
    try:
        pd = DaeProblemDef(shape, 1e-3)
        rng = np.random.default_rng(7)
        u = rng.standard_normal(pd.dim)
        w = rng.standard_normal(pd.dim)
        lu, _, gu, gw = pd.blocks_csr(u, w, 0.0)
        # the engine's slab axis is y (x fastest): shape (nx, ny) -> planes = ny
        sshape = (shape[0], shape[1])
        x = rng.standard_normal(pd.dim)
        ok_lu = np.allclose(SlabOperator(lu, sshape, rank, nranks)(scatter(x, sshape, rank,
                                                                          nranks).copy()),
                            scatter(lu @ x, sshape, rank, nranks), atol=1e-10)
        ok_gw = np.allclose(SlabOperator(gw, sshape, rank, nranks)(scatter(x, sshape, rank,
                                                                          nranks).copy()),
                            scatter(gw @ x, sshape, rank, nranks), atol=1e-12)
        c = rng.standard_normal(pd.dim)
        p0, nl = slab_range(shape[1], rank, nranks)
        padded = np.zeros(pd.dim)
        padded[p0 * shape[0]:(p0 + nl) * shape[0]] = scatter(c, sshape, rank, nranks)
        cg = _allreduce(padded)
        exact_gather = bool(np.array_equal(cg, c))
        y_loc = scatter(spla.spsolve(gw.tocsc(), cg), sshape, rank, nranks)
        parts = [None] * nranks
        dist.all_gather_object(parts, y_loc)
        if rank == 0:
            y_ref = spla.spsolve(gw.tocsc(), c)
            rel = float(np.linalg.norm(gather(parts, sshape) - y_ref) / np.linalg.norm(y_ref))
            queue.put((bool(ok_lu), bool(ok_gw), exact_gather, rel))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_dae_slabs_and_gathered_constraint_solve():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dae_worker, args=(r, 2, port, (12, 14), q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    ok_lu, ok_gw, exact_gather, rel = res
    assert ok_lu and ok_gw
    assert exact_gather
    assert rel <= 1e-13, rel


def _pencil_worker(rank, nranks, port, shape, queue):
    """The slab -> pencil transpose FFT of the constraint solve
    (csrc/dae.cu constraint_solve_slab) restated with numpy FFTs and a gloo
    all-to-all: rows transformed on the slabs, padded blocks exchanged, the y
    transforms and the eigenvalue division on pencils, and back; the zero-mean
    shift and the pinned row through two small all-reduces.  Compared with the
    global sparse solve of the reference's constraint matrix."""
    import scipy.sparse.linalg as spla

    from oracle.problems import DaeProblemDef

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=nranks)
    try:
        nx, ny = shape
        pd = DaeProblemDef(shape, 1e-3)
        rng = np.random.default_rng(11)
        u = rng.standard_normal(pd.dim)
        w = rng.standard_normal(pd.dim)
        _, _, _, gw = pd.blocks_csr(u, w, 0.0)
        c = rng.standard_normal(pd.dim)
        sigma = 0.7
        h2 = (1.0 / nx) * (1.0 / ny)
        ih2 = (nx * nx, ny * ny)
        p0, nl = slab_range(ny, rank, nranks)
        cl = scatter(c, shape, rank, nranks).copy()
        pin = p0 == 0
        C_, nylmax, cols = pencil_layout(nx, ny, nranks)
        nxh = nx // 2 + 1
        inv = 1.0 / (sigma * h2)
        f = inv * cl
        part = np.array([f.sum() - (f[0] if pin else 0.0), cl[0] if pin else 0.0])
        tot = _allreduce(part)
        if pin:
            f[0] = -tot[0]
        F = np.fft.rfft(f.reshape(nl, nx), axis=1)                  # (nl, nxh)
        send = np.zeros((nranks, nylmax, C_), dtype=complex)
        for d in range(nranks):
            k0 = d * C_
            send[d, :nl, :cols[d]] = F[:, k0:k0 + cols[d]]
        recv = np.zeros_like(send)
        ts, tr = torch.from_numpy(send.view(np.float64).reshape(-1)), \
            torch.from_numpy(recv.view(np.float64).reshape(-1))
        dist.all_to_all_single(tr, ts)
        lines = np.zeros((C_, ny), dtype=complex)
        for s_ in range(nranks):
            q0, ql = slab_range(ny, s_, nranks)
            lines[:cols[rank], q0:q0 + ql] = recv[s_, :ql, :cols[rank]].T
        L = np.fft.fft(lines[:cols[rank]], axis=1)
        kx = rank * C_ + np.arange(cols[rank])[:, None]
        ky = np.arange(ny)[None, :]
        lam = -4.0 * ih2[0] * np.sin(np.pi * kx / nx) ** 2 - 4.0 * ih2[1] * np.sin(np.pi * ky / ny) ** 2
        with np.errstate(divide="ignore"):
            scale = np.where((kx == 0) & (ky == 0), 0.0, 1.0 / lam)
        lines[:cols[rank]] = np.fft.ifft(L * scale, axis=1)
        for d in range(nranks):
            q0, ql = slab_range(ny, d, nranks)
            send[d] = 0.0
            send[d, :ql, :cols[rank]] = lines[:cols[rank], q0:q0 + ql].T
        dist.all_to_all_single(tr, ts)
        for s_ in range(nranks):
            k0 = s_ * C_
            F[:, k0:k0 + cols[s_]] = recv[s_, :nl, :cols[s_]]
        yt = np.fft.irfft(F, n=nx, axis=1).reshape(-1)
        yt0 = _allreduce(np.array([yt[0] if pin else 0.0]))[0]
        y_loc = (yt - yt0) + tot[1] / sigma
        parts = [None] * nranks
        dist.all_gather_object(parts, y_loc)
        if rank == 0:
            y_ref = spla.spsolve((sigma * gw).tocsc(), c)
            rel = float(np.linalg.norm(gather(parts, shape) - y_ref) / np.linalg.norm(y_ref))
            queue.put(rel)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("nranks,shape", [(2, (12, 14)), (3, (16, 10)), (3, (6, 7))])
def test_gloo_pencil_transpose_constraint_solve(nranks, shape):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pencil_worker, args=(r, nranks, port, shape, q))
             for r in range(nranks)]
    for p in procs:
        p.start()
    rel = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert rel <= 1e-12, rel


def test_pencil_layout_covers_the_half_spectrum():
    for nx, ny, p in [(2048, 2048, 8), (40, 40, 2), (32, 36, 3), (6, 7, 3), (10, 4, 8)]:
        c, nylmax, cols = pencil_layout(nx, ny, p)
        assert sum(cols) == nx // 2 + 1
        assert all(0 <= k <= c for k in cols)
        assert nylmax >= max(slab_range(ny, r, p)[1] for r in range(p))
