"""Row-distributed solve on one GPU: N ranks emulated inside
libpmgr (loopback transport, one host thread per rank, every exchange an
ordinary stream-ordered copy).  Bar: a distributed MGR application is
BITWISE equal to the single-GPU one (each local row sums its columns in the
global stored order with the global lane group / block layout), and the
distributed GMRES converges in the single-GPU iteration count +-1 to the same
solution."""

import numpy as np
import pytest

from tests.test_gpu_parity import mgr_config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pk():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1904_05960_b200 import amg, dist, krylov, mgr, problems, sparse

    return sparse, amg, mgr, krylov, dist, problems


def build(pk, pb, n_max=4, four=False):
    sparse, amg, mgr, krylov, dist, problems = pk
    A = sparse.CsrMatrix(pb.n, pb.n, pb.row_offsets, pb.col_indices, pb.values)
    h = mgr.mgr_setup(A, sparse.FieldLayout(pb.field_of, pb.entity_of), mgr_config(pk[:4], pb, n_max, four))
    return A, h


CASES = [("C2", dict(n=8), 4, False), ("C1", dict(n=8), None, False), ("C4", dict(n=6), 4, True)]


@pytest.mark.parametrize("name,kw,n_max,four", CASES)
@pytest.mark.parametrize("nranks", [1, 2, 3])
def test_distributed_apply_is_bitwise(pk, name, kw, n_max, four, nranks):
    sparse, amg, mgr, krylov, dist, problems = pk
    pb, bounds = problems.rank_major(problems.make(name, seed=3, **kw), nranks)
    A, h = build(pk, pb, n_max, four)
    v = np.random.default_rng(7).standard_normal(pb.n)
    z = h.apply(v)
    zd = dist.emulate_apply(h, bounds, v).cpu().numpy()
    assert np.array_equal(zd, z), f"max diff {np.abs(zd - z).max()}"


# the production configurations' multi-cycle AMG F-relaxation (C5: two
# V-cycles, C4: three) on the row-distributed path
PROD_CASES = [("C5", dict(nxy=8, nz_per_gpu=4, gpus=2)), ("C4", dict(n=6))]


@pytest.mark.parametrize("name,kw", PROD_CASES)
@pytest.mark.parametrize("nranks", [1, 2, 3])
def test_distributed_apply_production_is_bitwise(pk, name, kw, nranks):
    sparse, amg, mgr, krylov, dist, problems = pk
    pb, bounds = problems.rank_major(problems.make(name, seed=3, **kw), nranks)
    A = sparse.CsrMatrix(pb.n, pb.n, pb.row_offsets, pb.col_indices, pb.values)
    cfg = mgr.config_from_options(problems.solver_options(name, pb))
    assert max(lv.f_relax_sweeps for lv in cfg.levels) > 1
    h = mgr.mgr_setup(A, sparse.FieldLayout(pb.field_of, pb.entity_of), cfg)
    v = np.random.default_rng(7).standard_normal(pb.n)
    z = h.apply(v)
    zd = dist.emulate_apply(h, bounds, v).cpu().numpy()
    assert np.array_equal(zd, z), f"max diff {np.abs(zd - z).max()}"


@pytest.mark.parametrize("nranks", [2, 3])
def test_distributed_gmres_matches_oracle(pk, nranks):
    """The row-distributed GMRES (emulated ranks) against the CPU oracle on the
    same rank-major problem: iterations +-1, solution 1e-10 when the counts
    agree (the oracle is pinned to the reference, tests/test_oracle_golden.py)."""
    from oracle import oracle as O

    sparse, amg, mgr, krylov, dist, problems = pk
    pb, bounds = problems.rank_major(problems.make("C5", seed=4, nxy=10, nz_per_gpu=5, gpus=2), nranks)
    opts = problems.solver_options("C5", pb)
    A = sparse.CsrMatrix(pb.n, pb.n, pb.row_offsets, pb.col_indices, pb.values)
    h = mgr.mgr_setup(A, sparse.FieldLayout(pb.field_of, pb.entity_of), mgr.config_from_options(opts))
    cfg = krylov.GmresConfig(restart=opts["restart"], max_iters=opts["max_iters"], rtol=1e-6)
    xd, its, conv = dist.emulate_gmres(h, bounds, pb.rhs, cfg)
    xd = xd.cpu().numpy()
    oA = O.Csr(pb.n, pb.n, pb.row_offsets, pb.col_indices, pb.values)
    oh = O.mgr_setup(oA, pb.field_of, pb.entity_of, O.config_from_options(opts))
    xo, its_o, _, conv_o = O.gmres(lambda y: O.spmv(oA, y), oh.apply, pb.rhs, restart=opts["restart"],
                                   max_iters=opts["max_iters"], rtol=1e-6)
    rel = np.linalg.norm(xd - xo) / np.linalg.norm(xo)
    print(f"[dist {nranks}] iterations {its} (oracle {its_o}) solution rel {rel:.2e}")
    assert conv and conv_o and abs(its - its_o) <= 1
    assert rel <= (1e-10 if its == its_o else 1e-5), rel


def test_distributed_apply_uneven_and_empty_ranks(pk):
    """More ranks than some coarse spaces have rows: empty owned ranges."""
    sparse, amg, mgr, krylov, dist, problems = pk
    pb, bounds = problems.rank_major(problems.make("C2", seed=5, n=6), 6)
    A, h = build(pk, pb)
    v = np.random.default_rng(1).standard_normal(pb.n)
    assert np.array_equal(dist.emulate_apply(h, bounds, v).cpu().numpy(), h.apply(v))


def test_distributed_apply_original_layout_one_rank(pk):
    """One rank on the original (block-prefix) layout: the outer operator's
    block copy is sliced as CSR, the application stays bitwise."""
    sparse, amg, mgr, krylov, dist, problems = pk
    pb = problems.make("C2", seed=2, n=8)
    A, h = build(pk, pb)
    v = np.random.default_rng(3).standard_normal(pb.n)
    assert np.array_equal(dist.emulate_apply(h, [0, pb.n], v).cpu().numpy(), h.apply(v))


@pytest.mark.parametrize("nranks", [2, 4])
def test_distributed_gmres_matches_single_gpu(pk, nranks):
    sparse, amg, mgr, krylov, dist, problems = pk
    pb, bounds = problems.rank_major(problems.make("C2", seed=4, n=12), nranks)
    A, h = build(pk, pb)
    cfg = krylov.GmresConfig(restart=100, max_iters=400, rtol=1e-6)
    x1, st = krylov.gmres(A, h.apply, pb.rhs, cfg=cfg)
    xd, its, conv = dist.emulate_gmres(h, bounds, pb.rhs, cfg)
    xd = xd.cpu().numpy()
    assert conv and st.converged
    assert abs(its - st.iterations) <= 1
    r = pb.rhs - sparse.matvec(A, xd)
    assert np.linalg.norm(r) <= 1e-6 * np.linalg.norm(pb.rhs) * (1 + 1e-9)
    assert np.linalg.norm(xd - x1) <= 1e-5 * np.linalg.norm(x1)


def test_single_rank_solver_api(pk):
    """The per-rank API (what a torchrun job calls) with one rank."""
    sparse, amg, mgr, krylov, dist, problems = pk
    pb, bounds = problems.rank_major(problems.make("C2", seed=6, n=8), 1)
    A, h = build(pk, pb)
    d = dist.DeviceDistSolver(h, bounds, 0, 1)
    assert (d.lo, d.n_own) == (0, pb.n)
    v = np.random.default_rng(2).standard_normal(pb.n)
    assert np.array_equal(d.apply(v).cpu().numpy(), h.apply(v))
    y = d.spmv(v).cpu().numpy()
    assert np.allclose(y, sparse.matvec(A, v), rtol=1e-13, atol=1e-13 * np.abs(y).max())
    x, st = d.gmres(pb.rhs, krylov.GmresConfig(restart=100, max_iters=300))
    assert st.converged
    r = pb.rhs - sparse.matvec(A, x.cpu().numpy())
    assert np.linalg.norm(r) <= 1e-6 * np.linalg.norm(pb.rhs) * (1 + 1e-9)


def test_distribution_rejects_unsupported(pk):
    sparse, amg, mgr, krylov, dist, problems = pk
    pb, bounds = problems.rank_major(problems.make("C2", seed=1, n=6), 2)
    A, h = build(pk, pb)
    with pytest.raises(ValueError):
        dist.emulate_apply(h, [0, 5, pb.n - 1], np.zeros(pb.n))  # bounds do not cover [0, n)


def test_nccl_transport_single_rank(pk):
    """The NCCL transport (libnccl resolved at run time) on a one-rank
    communicator: id, communicator, grouped send/recv, all-reduce."""
    sparse, amg, mgr, krylov, dist, problems = pk
    pb, bounds = problems.rank_major(problems.make("C2", seed=8, n=8), 1)
    A, h = build(pk, pb)
    tr = dist.nccl_transport(0, 1, None)
    d = dist.DeviceDistSolver(h, bounds, 0, 1, tr)
    v = np.random.default_rng(4).standard_normal(pb.n)
    assert np.array_equal(d.apply(v).cpu().numpy(), h.apply(v))
    x, st = d.gmres(pb.rhs, krylov.GmresConfig(restart=100, max_iters=300))
    x1, st1 = krylov.gmres(A, h.apply, pb.rhs, cfg=krylov.GmresConfig(restart=100, max_iters=300))
    assert st.converged and abs(st.iterations - st1.iterations) <= 1


_LONG_ROWS_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from tests.test_gpu_dist import build
from paper_1904_05960_b200 import amg, dist, krylov, mgr, problems, sparse
pk = (sparse, amg, mgr, krylov, dist, problems)
pb, bounds = problems.rank_major(problems.make("C4", seed=3, n=14), 3)
A, h = build(pk, pb, 4, True)
v = np.random.default_rng(7).standard_normal(pb.n)
z = h.apply(v)
zd = dist.emulate_apply(h, bounds, v).cpu().numpy()
print("BITWISE", bool(np.array_equal(zd, z)), float(np.abs(zd - z).max()))
"""


def test_distributed_apply_bitwise_with_long_rows(pk, tmp_path):
    """Coarse AMG levels kept sparse (collapse threshold 300 rows) so that
    skewed operators with block-per-row long rows reach the distributed
    cycle: every rank's slice takes the same path per row as the global
    operator, so the application stays bitwise equal."""
    import os
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PMGR_COLLAPSE_ROWS="300", PMGR_HIER_STATS="1")
    r = subprocess.run([sys.executable, "-c", _LONG_ROWS_SCRIPT, repo], env=env, capture_output=True, text=True,
                       timeout=600, cwd=repo)
    assert r.returncode == 0, r.stderr[-2000:]
    longs = [ln for ln in r.stderr.splitlines() if "long rows" in ln and "long rows 0 " not in ln]
    assert longs, "no operator exercised the long-row path"
    assert "BITWISE True" in r.stdout, r.stdout


_DIST_SETUP_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from tests.test_gpu_dist import build
from tests.test_gpu_parity import mgr_config
from paper_1904_05960_b200 import amg, dist, krylov, mgr, problems, sparse
pk = (sparse, amg, mgr, krylov, dist, problems)
for name, n, n_max, four in (("C2", 12, 4, False), ("C1", 12, None, False), ("C4", 10, 4, True), ("C4p", 10, 4, True)):
    for nranks in (1, 2, 3):
        pb, bounds = problems.rank_major(problems.make(name[:2], seed=3, n=n), nranks)
        if name == "C4p":  # production configuration: three AMG V-cycles of F-relaxation
            cfg = mgr.config_from_options(problems.solver_options("C4", pb))
            A = sparse.CsrMatrix(pb.n, pb.n, pb.row_offsets, pb.col_indices, pb.values)
            h = mgr.mgr_setup(A, sparse.FieldLayout(pb.field_of, pb.entity_of), cfg)
        else:
            A, h = build(pk, pb, n_max, four)
            cfg = mgr_config(pk[:4], pb, n_max, four)
        lay = sparse.FieldLayout(pb.field_of, pb.entity_of)
        v = np.random.default_rng(7).standard_normal(pb.n)
        z = h.apply(v)
        zd = dist.emulate_setup_apply(A, lay, cfg, bounds, v).cpu().numpy()
        print("CASE", name, nranks, "BITWISE", bool(np.array_equal(zd, z)), float(np.abs(zd - z).max()))
        x, its, conv = dist.emulate_setup_gmres(A, lay, cfg, bounds, pb.rhs, krylov.GmresConfig(restart=100, max_iters=500))
        xs, st = krylov.gmres(A, h.apply, pb.rhs, cfg=krylov.GmresConfig(restart=100, max_iters=500))
        print("GMRES", name, nranks, its, st.iterations, conv, float(np.linalg.norm(x.cpu().numpy() - xs) / np.linalg.norm(xs)))
"""


def test_distributed_setup_is_bitwise():
    """The distributed setup (every rank sets up the owned rows of every
    operator from its row slice: MIS rounds with status exchanges, transposes
    assembled at their owners, Galerkin products over fetched ghost rows,
    small levels gathered) gives a hierarchy whose distributed application is
    bitwise equal to the single-GPU one, and a distributed GMRES within +-1
    iteration.  Coarse levels are kept distributed down to 300 rows
    (PMGR_COLLAPSE_ROWS / PMGR_DIST_REPLICATE_ROWS) so that the small test
    problems exercise several distributed AMG levels."""
    import os
    import subprocess
    import sys

    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PMGR_COLLAPSE_ROWS="300", PMGR_DIST_REPLICATE_ROWS="300")
    r = subprocess.run([sys.executable, "-c", _DIST_SETUP_SCRIPT, repo], env=env, capture_output=True, text=True,
                       timeout=900, cwd=repo)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    cases = [ln.split() for ln in r.stdout.splitlines() if ln.startswith("CASE")]
    assert len(cases) == 12, r.stdout
    bad = [c for c in cases if c[4] != "True"]
    assert not bad, r.stdout
    for ln in r.stdout.splitlines():
        if ln.startswith("GMRES"):
            _, name, nr, its, its1, conv, rel = ln.split()
            assert conv == "True" and abs(int(its) - int(its1)) <= 1 and float(rel) < 1e-5, ln


_OVERLAP_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_1904_05960_b200 import dist, mgr, problems, sparse
for name, base in (("C5", problems.make_c5(seed=3, nxy=10, nz_per_gpu=6, gpus=3)), ("C4", problems.make_c4(seed=3, n=12))):
    pb, bounds = problems.rank_major(base, 3)
    A = sparse.CsrMatrix(pb.n, pb.n, pb.row_offsets, pb.col_indices, pb.values)
    h = mgr.mgr_setup(A, sparse.FieldLayout(pb.field_of, pb.entity_of),
                      mgr.config_from_options(problems.solver_options(name, pb)))
    v = np.random.default_rng(7).standard_normal(pb.n)
    print("BITWISE", name, bool(np.array_equal(dist.emulate_apply(h, bounds, v).cpu().numpy(), h.apply(v))))
"""


def test_halo_overlap_split_is_bitwise(pk):
    """Row-distributed operators split into interior and boundary row ranges
    (the interior rows run while the halo exchange is in flight): the split
    is taken (PMGR_HIER_STATS reports it) and the application stays bitwise
    equal to the single-GPU one, with the overlap on and off."""
    import os
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for ov in ("1", "0"):
        env = dict(os.environ, PMGR_HIER_STATS="1", PMGR_OVERLAP=ov)
        r = subprocess.run([sys.executable, "-c", _OVERLAP_SCRIPT, repo], env=env, capture_output=True, text=True,
                           timeout=600, cwd=repo)
        assert r.returncode == 0, r.stderr[-3000:]
        outs[ov] = r
        assert r.stdout.count("BITWISE") == 2 and "False" not in r.stdout, r.stdout
    splits = [ln for ln in outs["1"].stderr.splitlines() if "overlap split" in ln]
    assert any("outer 0 " not in ln for ln in splits), "no operator has boundary rows"


def test_distributed_apply_bitwise_with_sliced_jagged_copies(pk):
    """A problem large enough for the sliced jagged solve copies at their
    DEFAULT thresholds (C4 at 44^3: A0, the displacement block and A_CF take
    them): the rank-local slices carry the copies the global operators take
    (same lanes per row, same order), so the distributed application -- of
    the sliced hierarchy and of the distributed setup -- stays bitwise equal
    to the single-GPU one, interior / boundary row ranges included."""
    sparse, amg, mgr, krylov, dist, problems = pk
    pb, bounds = problems.rank_major(problems.make("C4", seed=3, n=44), 2)
    A = sparse.CsrMatrix(pb.n, pb.n, pb.row_offsets, pb.col_indices, pb.values)
    lay = sparse.FieldLayout(pb.field_of, pb.entity_of)
    cfg = mgr.config_from_options(problems.solver_options("C4", pb))
    h = mgr.mgr_setup(A, lay, cfg)
    v = np.random.default_rng(7).standard_normal(pb.n)
    z = h.apply(v)
    zd = dist.emulate_apply(h, bounds, v).cpu().numpy()
    assert np.array_equal(zd, z), f"sliced hierarchy: max diff {np.abs(zd - z).max()}"
    zs = dist.emulate_setup_apply(A, lay, cfg, bounds, v).cpu().numpy()
    assert np.array_equal(zs, z), f"distributed setup: max diff {np.abs(zs - z).max()}"


@pytest.mark.parametrize("name,kw", [("C5", dict(nxy=10, nz_per_gpu=5, gpus=2)), ("C4", dict(n=8))])
@pytest.mark.parametrize("variant", ["parity", "production"])
def test_distributed_setup_bitwise_at_default_thresholds(pk, name, kw, variant):
    """At the DEFAULT replication / collapse thresholds the whole F-relaxation
    AMG of these small problems is gathered and set up on every rank; the
    gathered displacement block keeps its 3x3 block copy, so the distributed
    setup's application is bitwise the single-GPU one (it differed by 4e-13
    while the gathered level ran on the CSR kernels)."""
    sparse, amg, mgr, krylov, dist, problems = pk
    pb, bounds = problems.rank_major(problems.make(name, seed=4, **kw), 2)
    A = sparse.CsrMatrix(pb.n, pb.n, pb.row_offsets, pb.col_indices, pb.values)
    lay = sparse.FieldLayout(pb.field_of, pb.entity_of)
    cfg = mgr.config_from_options(problems.solver_options(name, pb, variant=variant))
    h = mgr.mgr_setup(A, lay, cfg)
    v = np.random.default_rng(11).standard_normal(pb.n)
    z = h.apply(v)
    zs = dist.emulate_setup_apply(A, lay, cfg, bounds, v).cpu().numpy()
    assert np.array_equal(zs, z), f"max diff {np.abs(zs - z).max()}"


@pytest.mark.parametrize("nranks", [1, 2, 3])
def test_distributed_ilu_smoother_level_is_bitwise(pk, nranks):
    """C3's production configuration (ILU(1) global smoother over partitions
    of 16 flow rows on the second level) row-distributed: the partitions fall
    on the z-slab boundaries, every rank applies the global factors of its
    own partitions and exchanges the smoothed iterate's ghosts before the
    level operator and its C rows read it -- bitwise the single-GPU
    application, and the distributed GMRES converges like the single-GPU one."""
    sparse, amg, mgr, krylov, dist, problems = pk
    pb, bounds = problems.rank_major(problems.make("C3", seed=3, n=8), nranks)
    A = sparse.CsrMatrix(pb.n, pb.n, pb.row_offsets, pb.col_indices, pb.values)
    opts = problems.solver_options("C3", pb)
    cfg = mgr.config_from_options(opts)
    assert any(lv.global_smoother == "ilu" for lv in cfg.levels)
    h = mgr.mgr_setup(A, sparse.FieldLayout(pb.field_of, pb.entity_of), cfg)
    v = np.random.default_rng(7).standard_normal(pb.n)
    z = h.apply(v)
    zd = dist.emulate_apply(h, bounds, v).cpu().numpy()
    assert np.array_equal(zd, z), f"max diff {np.abs(zd - z).max()}"
    gcfg = krylov.GmresConfig(restart=opts["restart"], max_iters=2000, rtol=1e-8)
    x1, st = krylov.gmres(A, h.apply, pb.rhs, cfg=gcfg)
    xd, its, conv = dist.emulate_gmres(h, bounds, pb.rhs, gcfg)
    assert st.converged and conv and abs(its - st.iterations) <= 1, (its, st.iterations)
    xd = xd.cpu().numpy()
    assert np.linalg.norm(xd - x1) <= 1e-6 * np.linalg.norm(x1)
