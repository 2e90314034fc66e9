"""z-slab decomposition on CPU with world_size 2 (gloo): ownership, halo
plans, distributed SpMV and distributed GMRES against the global oracle.
The local compute here is the oracle (test infrastructure); on the GPU the
same plumbing drives libpmgr's kernels over NCCL."""

import os
import socket
import sys
import tempfile

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, outdir):
    sys.path.insert(0, REPO)
    import torch
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_1904_05960_b200 import dist as D
    from paper_1904_05960_b200 import problems

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    pb = problems.make_c2(seed=4, n=6)
    owner = D.dof_owner(pb, world)
    plan = D.build_halo_plan(pb.row_offsets, pb.col_indices, pb.values, owner, rank, world)
    local = O.Csr(plan.n_own, plan.n_ext, plan.ro, plan.ci, plan.v)

    def local_matvec(x_ext):
        return torch.from_numpy(O.spmv(local, x_ext.numpy()))

    op = D.DistOperator(plan, local_matvec, dist)
    x = np.random.default_rng(0).standard_normal(pb.n)
    y_own = op(torch.from_numpy(x[plan.owned].copy())).numpy()
    # Jacobi preconditioner from the owned diagonal
    A = O.Csr(pb.n, pb.n, pb.row_offsets, pb.col_indices, pb.values)
    dinv = torch.from_numpy(1.0 / A.diagonal()[plan.owned])
    b = torch.from_numpy(pb.rhs[plan.owned].copy())
    xs, its, hist, conv = D.dist_gmres(op, lambda v: dinv * v, b, dist, restart=40, max_iters=400, rtol=1e-8)
    np.savez(os.path.join(outdir, f"r{rank}.npz"), owned=plan.owned, ghosts=plan.ghosts, y=y_own, x=xs.numpy(),
             its=its, conv=conv, hist=hist, nsend=sum(len(v) for v in plan.send_to.values()),
             nrecv=sum(len(v) for v in plan.recv_from.values()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.fixture(scope="module")
def run2():
    import torch.multiprocessing as mp

    outdir = tempfile.mkdtemp()
    mp.spawn(_worker, args=(2, _free_port(), outdir), nprocs=2, join=True)
    return [dict(np.load(os.path.join(outdir, f"r{r}.npz"))) for r in range(2)]


def test_slab_partition_covers_every_dof_once():
    from paper_1904_05960_b200 import dist as D
    from paper_1904_05960_b200 import problems

    pb = problems.make_c2(seed=4, n=6)
    for world in (1, 2, 3, 6):
        owner = D.dof_owner(pb, world)
        assert owner.min() == 0 and owner.max() == world - 1
        counts = np.bincount(owner, minlength=world)
        assert counts.sum() == pb.n and np.all(counts > 0)
    with pytest.raises(ValueError):
        D.slab_bounds(4, 5)


def test_halo_plans_are_consistent():
    from paper_1904_05960_b200 import dist as D
    from paper_1904_05960_b200 import problems

    pb = problems.make_c4(seed=1, n=4)
    world = 3
    owner = D.dof_owner(pb, world)
    plans = [D.build_halo_plan(pb.row_offsets, pb.col_indices, pb.values, owner, r, world) for r in range(world)]
    for p in plans:
        assert np.all(owner[p.ghosts] != p.rank)
        for peer, idx in p.recv_from.items():
            # what I receive from peer is exactly what peer sends to me, in the same order
            sent = plans[peer].owned[plans[peer].send_to[p.rank]]
            assert np.array_equal(p.ghosts[idx], sent)
        # slabs only talk to z-neighbours
        assert set(p.recv_from) <= {p.rank - 1, p.rank + 1}


def test_distributed_spmv_is_bitwise_global(run2):
    from oracle import oracle as O
    from paper_1904_05960_b200 import problems

    pb = problems.make_c2(seed=4, n=6)
    A = O.Csr(pb.n, pb.n, pb.row_offsets, pb.col_indices, pb.values)
    x = np.random.default_rng(0).standard_normal(pb.n)
    y = O.spmv(A, x)
    for res in run2:
        assert np.array_equal(res["y"], y[res["owned"]])
        assert res["nsend"] > 0 and res["nrecv"] > 0


def test_distributed_gmres_matches_global(run2):
    from oracle import oracle as O
    from paper_1904_05960_b200 import problems

    pb = problems.make_c2(seed=4, n=6)
    A = O.Csr(pb.n, pb.n, pb.row_offsets, pb.col_indices, pb.values)
    dinv = 1.0 / A.diagonal()
    xg, its, hist, conv = O.gmres(lambda v: O.spmv(A, v), lambda v: dinv * v, pb.rhs, restart=40, max_iters=400,
                                  rtol=1e-8)
    assert run2[0]["its"] == run2[1]["its"]
    assert abs(int(run2[0]["its"]) - its) <= 1
    x = np.zeros(pb.n)
    for res in run2:
        x[res["owned"]] = res["x"]
    assert np.linalg.norm(x - xg) <= 1e-6 * np.linalg.norm(xg)
    assert bool(run2[0]["conv"]) == conv


@pytest.mark.parametrize("nranks", [1, 2, 3, 5])
def test_rank_major_numbering(nranks):
    """problems.rank_major: a symmetric renumbering P A P^T whose rank ranges
    are exactly the z-slab ownership of `dof_owner`, valid CSR (sorted
    columns), identity for one rank (the layout libpmgr's row distribution
    slices)."""
    import scipy.sparse as sp

    from paper_1904_05960_b200 import dist as D
    from paper_1904_05960_b200 import problems

    pb = problems.make_c2(seed=2, n=5)
    q, bounds = problems.rank_major(pb, nranks)
    perm = q.meta["perm"]
    assert bounds[0] == 0 and bounds[-1] == pb.n and np.all(np.diff(bounds) > 0)
    owner = D.dof_owner(pb, nranks)
    for r in range(nranks):
        assert np.all(owner[perm[bounds[r]:bounds[r + 1]]] == r)
    A = sp.csr_matrix((pb.values, pb.col_indices, pb.row_offsets), shape=(pb.n, pb.n))
    B = sp.csr_matrix((q.values, q.col_indices, q.row_offsets), shape=(q.n, q.n))
    assert abs(A[perm][:, perm] - B).max() == 0.0
    for i in range(0, q.n, 97):
        cols = q.col_indices[q.row_offsets[i]:q.row_offsets[i + 1]]
        assert np.all(np.diff(cols) > 0)
    assert np.array_equal(q.field_of, pb.field_of[perm]) and np.array_equal(q.rhs, pb.rhs[perm])
    if nranks == 1:
        assert np.array_equal(perm, np.arange(pb.n))
        assert np.array_equal(q.col_indices, pb.col_indices) and np.array_equal(q.values, pb.values)


# ---------------------------------------------------------------------------
# distributed setup of one AMG level (the algorithm of csrc/dsetup.cu, here
# with the oracle's kernels and gloo): owned rows in the global row space,
# S^T assembled at the owners, MIS rounds with status all-gathers, R = P^T
# assembled at the coarse owners, Galerkin over fetched ghost rows.

def _rows(M, lo, hi):
    from oracle import oracle as O

    ro = np.clip(M.ro, M.ro[lo], M.ro[hi]) - M.ro[lo]
    return O.Csr(M.nrows, M.ncols, ro, M.ci[M.ro[lo]:M.ro[hi]], M.v[M.ro[lo]:M.ro[hi]])


def _with_rows(M, extra):
    """M (partial, global row space) plus {row: (cols, vals)} rows."""
    from oracle import oracle as O

    lens = np.diff(M.ro).copy()
    for r, (c, v) in extra.items():
        lens[r] = len(c)
    ro = np.concatenate([[0], np.cumsum(lens)])
    ci = np.empty(ro[-1], dtype=np.int32)
    v = np.empty(ro[-1])
    for r in range(M.nrows):
        if r in extra:
            ci[ro[r]:ro[r + 1]], v[ro[r]:ro[r + 1]] = extra[r]
        else:
            ci[ro[r]:ro[r + 1]], v[ro[r]:ro[r + 1]] = M.ci[M.ro[r]:M.ro[r + 1]], M.v[M.ro[r]:M.ro[r + 1]]
    return O.Csr(M.nrows, M.ncols, ro, ci, v)


def _fetch(dist, M, want, start, world):
    """rows `want` of the row-distributed M from their owners"""
    reqs = [None] * world
    dist.all_gather_object(reqs, sorted(set(int(w) for w in want)))
    mine = {}
    for p, rq in enumerate(reqs):
        mine[p] = {r: (M.ci[M.ro[r]:M.ro[r + 1]].copy(), M.v[M.ro[r]:M.ro[r + 1]].copy())
                   for r in rq if start[dist.get_rank()] <= r < start[dist.get_rank() + 1]}
    got = [None] * world
    dist.all_gather_object(got, mine)
    out = {}
    for p in range(world):
        out.update(got[p][dist.get_rank()])
    return out


def _setup_worker(rank, world, port, outdir):
    sys.path.insert(0, REPO)
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_1904_05960_b200 import problems

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    pb, bounds = problems.rank_major(problems.make_c2(seed=4, n=6), world)
    A = O.Csr(pb.n, pb.n, pb.row_offsets, pb.col_indices, pb.values)
    isu = pb.field_of == 0
    Auu = O.extract_blocks(A, ~isu)[0]
    nu = Auu.nrows
    ust = [int(isu[:b].sum()) for b in bounds]
    lo, hi = ust[rank], ust[rank + 1]
    funcs = np.arange(nu) % 3
    Ap = _rows(Auu, lo, hi)
    mask = O.strength_mask(Ap, 0.5, funcs)
    S = O.mask_to_pattern(Ap, mask)
    # S^T: strong pairs (i, j) sent to the owner of j
    i_of, j_of = S.rows_of_entries(), S.ci.astype(np.int64)
    pieces = [None] * world
    dist.all_gather_object(pieces, {q: (i_of[(j_of >= ust[q]) & (j_of < ust[q + 1])],
                                        j_of[(j_of >= ust[q]) & (j_of < ust[q + 1])]) for q in range(world)})
    ins = [[] for _ in range(hi - lo)]
    for p in range(world):
        ii, jj = pieces[p][rank]
        for i, j in zip(ii, jj):
            ins[j - lo].append(int(i))
    segs = [None] * world
    dist.all_gather_object(segs, np.array([len(x) for x in ins], dtype=np.int64))
    meas = np.concatenate(segs)
    # lexicographically-first MIS rounds on the owned points
    status = np.zeros(nu, dtype=np.int8)
    rounds = 0
    while True:
        rounds += 1
        new = status[lo:hi].copy()
        for v in range(lo, hi):
            if status[v]:
                continue
            nb = list(S.ci[S.ro[v]:S.ro[v + 1]]) + ins[v - lo]
            early = [u for u in nb if meas[u] > meas[v] or (meas[u] == meas[v] and u < v)]
            if any(status[u] == 1 for u in early):
                new[v - lo] = 2
            elif all(status[u] == 2 for u in early):
                new[v - lo] = 1
        segs = [None] * world
        dist.all_gather_object(segs, new)
        status = np.concatenate(segs)
        if not (status == 0).any():
            break
    is_c = status == 1
    cst = [int(is_c[:u].sum()) for u in ust]
    # interpolation is row-local: the owned rows of P
    Pg, _ = O.direct_interpolation(Auu, O.strength_mask(Auu, 0.5, funcs), is_c, funcs)
    Pp = _rows(Pg, lo, hi)
    # R = P^T: my fine rows' entries assembled at the coarse owners, rank order
    Rt = O.transpose(Pp)
    parts = [None] * world
    dist.all_gather_object(parts, {q: {c: (Rt.ci[Rt.ro[c]:Rt.ro[c + 1]].copy(), Rt.v[Rt.ro[c]:Rt.ro[c + 1]].copy())
                                       for c in range(cst[q], cst[q + 1])} for q in range(world)})
    R_rows = {}
    for c in range(cst[rank], cst[rank + 1]):
        cs = [parts[p][rank][c] for p in range(world)]
        R_rows[c] = (np.concatenate([x[0] for x in cs]), np.concatenate([x[1] for x in cs]))
    nc = int(is_c.sum())
    R = _with_rows(O.Csr(nc, nu, np.zeros(nc + 1, dtype=np.int64), np.zeros(0, np.int32), np.zeros(0)), R_rows)
    want = [c for c in np.unique(R.ci) if not lo <= c < hi]
    T1 = O.spgemm(R, _with_rows(Ap, _fetch(dist, Ap, want, ust, world)), False)
    want = [c for c in np.unique(T1.ci) if not lo <= c < hi]
    Ac = O.spgemm(T1, _with_rows(Pp, _fetch(dist, Pp, want, ust, world)), False)
    np.savez(os.path.join(outdir, f"s{rank}.npz"), is_c=is_c, rounds=rounds, clo=cst[rank], chi=cst[rank + 1],
             ro=Ac.ro, ci=Ac.ci, v=Ac.v)
    dist.barrier()
    dist.destroy_process_group()


def test_distributed_amg_level_setup_matches_global():
    """world_size 2 (gloo): the distributed coarsening reproduces the
    reference's sequential greedy MIS exactly, and the owned rows of the
    distributed Galerkin product P^T A P are bitwise the global rows."""
    import torch.multiprocessing as mp

    from oracle import oracle as O
    from paper_1904_05960_b200 import problems

    outdir = tempfile.mkdtemp()
    mp.spawn(_setup_worker, args=(2, _free_port(), outdir), nprocs=2, join=True)
    res = [dict(np.load(os.path.join(outdir, f"s{r}.npz"))) for r in range(2)]
    pb, _ = problems.rank_major(problems.make_c2(seed=4, n=6), 2)
    A = O.Csr(pb.n, pb.n, pb.row_offsets, pb.col_indices, pb.values)
    Auu = O.extract_blocks(A, pb.field_of != 0)[0]
    funcs = np.arange(Auu.nrows) % 3
    mask = O.strength_mask(Auu, 0.5, funcs)
    is_c = O.greedy_mis(O.mask_to_pattern(Auu, mask))
    P, _ = O.direct_interpolation(Auu, mask, is_c, funcs)
    Ac = O.galerkin(P, O.transpose(P), Auu)
    for r in res:
        assert np.array_equal(r["is_c"], is_c)
        lo, hi = int(r["clo"]), int(r["chi"])
        assert np.array_equal(np.diff(r["ro"])[lo:hi], np.diff(Ac.ro)[lo:hi])
        a, b = Ac.ro[lo], Ac.ro[hi]
        assert np.array_equal(r["ci"], Ac.ci[a:b]) and np.array_equal(r["v"], Ac.v[a:b])
    assert int(res[0]["rounds"]) >= 2
