"""On-device Jacobian assembly: the device CSR equals the
host generator's (problems.assemble) bitwise for every configuration family,
and solves identically."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pk():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1904_05960_b200 import problems, sparse

    return problems, sparse


CASES = [("C1", dict(n=5)), ("C2", dict(n=6)), ("C3", dict(n=8)), ("C4", dict(n=4)),
         ("C5", dict(nxy=4, nz_per_gpu=3, gpus=2)), ("C2", dict(n=7))]


@pytest.mark.parametrize("name,kw", CASES)
def test_device_assembly_is_bitwise(pk, name, kw):
    problems, sparse = pk
    host = problems.make(name, seed=11, **kw)
    dev = problems.make(name, seed=11, device=True, **kw)
    H = dev.A.to_host()
    assert (H.nrows, H.ncols, H.nnz) == (host.n, host.n, host.nnz)
    assert np.array_equal(H.row_offsets, host.row_offsets)
    assert np.array_equal(H.col_indices, host.col_indices)
    assert np.array_equal(H.values, host.values), np.abs(H.values - host.values).max()
    assert np.array_equal(dev.field_of, host.field_of) and np.array_equal(dev.entity_of, host.entity_of)
    assert np.array_equal(dev.rhs, host.rhs)


def test_device_assembled_system_solves(pk):
    problems, sparse = pk
    from paper_1904_05960_b200 import amg, krylov, mgr

    dev = problems.make("C2", seed=2, n=8, device=True)
    F = sparse.Field
    cfg = mgr.MgrConfig(levels=(mgr.MgrLevelSpec({F.U}, {F.S, F.P}, f_relax="amg", n_max=4),
                                mgr.MgrLevelSpec({F.S}, {F.P}, f_relax="jacobi")),
                        amg_f_relax=amg.AmgConfig(strength_threshold=0.5, num_functions=3, npartitions=10 ** 9),
                        amg_terminal=amg.AmgConfig(strength_threshold=0.25, npartitions=10 ** 9))
    h = mgr.mgr_setup(dev.A, sparse.FieldLayout(dev.field_of, dev.entity_of), cfg)
    x, st = krylov.gmres(dev.A, h.apply, dev.rhs, cfg=krylov.GmresConfig(restart=100, max_iters=400))
    host = problems.make("C2", seed=2, n=8)
    A = sparse.CsrMatrix(host.n, host.n, host.row_offsets, host.col_indices, host.values)
    h2 = mgr.mgr_setup(A, sparse.FieldLayout(host.field_of, host.entity_of), cfg)
    x2, st2 = krylov.gmres(A, h2.apply, host.rhs, cfg=krylov.GmresConfig(restart=100, max_iters=400))
    assert st.converged and st.iterations == st2.iterations
    assert np.array_equal(x, x2)


@pytest.mark.parametrize("nranks", [1, 3])
def test_device_rank_major_matches_host(pk, nranks):
    problems, sparse = pk
    host, b1 = problems.rank_major(problems.make("C2", seed=4, n=6), nranks)
    dev, b2 = problems.rank_major(problems.make("C2", seed=4, n=6, device=True), nranks)
    assert np.array_equal(b1, b2)
    H = dev.A.to_host()
    assert np.array_equal(H.row_offsets, host.row_offsets)
    assert np.array_equal(H.col_indices, host.col_indices)
    assert np.array_equal(H.values, host.values)
    assert np.array_equal(dev.field_of, host.field_of) and np.array_equal(dev.rhs, host.rhs)
