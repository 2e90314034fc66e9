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
