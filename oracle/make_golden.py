"""Generate tests/golden/* by running the REFERENCE itself (poromgr).

Run in the build container only (the reference is not on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python oracle/make_golden.py

It imports /root/reference/pkg/src read-only, applies the two adapter shims
SURVEY.md §8c prescribes (FieldLayout.restrict downgrade for the mgr.py:359
interleave bug; a hand-built hierarchy for the 4-field config), configures
the parity smoother (npartitions >= n, i.e. l1-Jacobi) and dumps every setup
product, one preconditioner application and a GMRES solve.  Small cases are
stored as full arrays; large ones as SHA-256 digests of the canonical bytes
(zeros normalised to +0.0) plus the vectors.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = os.environ.get("POROMGR_SRC", "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
OUT = os.path.join(REPO, "tests", "golden")
sys.path.insert(0, REF)
sys.path.insert(0, REPO)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import numba  # noqa: E402
import scipy  # noqa: E402
import poromgr.sparse as psp  # noqa: E402

_orig_restrict = psp.FieldLayout.restrict


def _restrict(self, idx):  # shim 1: mgr.py:359 x sparse.py:180-189
    try:
        return _orig_restrict(self, idx)
    except ValueError:
        return psp.FieldLayout(self.field_of[idx], self.entity_of[idx], psp.Ordering.FIELD_BLOCKED)


psp.FieldLayout.restrict = _restrict

from poromgr import mgr as pmgr  # noqa: E402
from poromgr.amg import AmgConfig, amg_setup, amg_vcycle, strength_graph  # noqa: E402
from poromgr.krylov import GmresConfig, gmres  # noqa: E402
from poromgr.smoothers import PartitionSet, l1_diagonal, l1_gs_sweep  # noqa: E402
from poromgr.sparse import (CfSplitting, CsrMatrix, Field, FieldLayout, extract_blocks,  # noqa: E402
                            matvec, sparsify, spgemm, subtract)

from paper_1904_05960_b200 import problems  # noqa: E402

JACOBI = 10 ** 9
VERSIONS = dict(numpy=np.__version__, scipy=scipy.__version__, numba=numba.__version__)


def digest(ro, ci, v=None) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(ro, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(ci, dtype=np.int32).tobytes())
    if v is not None:
        vv = np.ascontiguousarray(v, dtype=np.float64) + 0.0
        h.update(vv.tobytes())
    return h.hexdigest()


def dcsr(m: CsrMatrix) -> str:
    return digest(m.row_offsets, m.col_indices, m.values)


def put_csr(d, key, m: CsrMatrix):
    d[key + "_ro"] = m.row_offsets
    d[key + "_ci"] = m.col_indices
    d[key + "_v"] = m.values
    d[key + "_shape"] = np.array(m.shape)


def parity_config(levels, f_parts=JACOBI, t_parts=JACOBI):
    return pmgr.MgrConfig(levels=levels,
                          amg_f_relax=AmgConfig(strength_threshold=0.5, num_functions=3, npartitions=f_parts),
                          amg_terminal=AmgConfig(strength_threshold=0.25, npartitions=t_parts))


def levels_for(pb, n_max):
    if pb.cell_fields == (problems.FIELD_P,):
        return (pmgr.MgrLevelSpec({Field.U}, {Field.P}, f_relax="amg", n_max=n_max),)
    return (pmgr.MgrLevelSpec({Field.U}, {Field.S, Field.P}, f_relax="amg", n_max=n_max),
            pmgr.MgrLevelSpec({Field.S}, {Field.P}, f_relax="jacobi", n_max=None))


def setup_4field(A, layout, n_max, cfg, opts=None):
    """Shim 2: U -> S2 -> S1 -> P built from reference primitives
    (mgr.py:300-326 containers).  `opts` (problems.
    solver_options) supplies the per-level F-relaxation sweeps and global
    smoothers; the spec objects only carry mode strings, so the S2 level is
    described to the reference as an S level."""
    cur, lay = A, layout
    levs = []
    tags = [problems.FIELD_U, problems.FIELD_S2, problems.FIELD_S]
    lvopts = opts["levels"] if opts else [dict(f_relax="amg", n_max=n_max), dict(f_relax="jacobi"),
                                          dict(f_relax="jacobi")]
    for tag, lo in zip(tags, lvopts):
        fspec = {Field.U} if tag == problems.FIELD_U else {Field.S}
        spec = pmgr.MgrLevelSpec(fspec, {Field.P}, f_relax=lo.get("f_relax", "jacobi"),
                                 f_relax_sweeps=lo.get("f_relax_sweeps", 1), n_max=lo.get("n_max"),
                                 global_smoother=lo.get("global_smoother", "none"))
        split = CfSplitting(lay.field_of != tag)
        blocks = extract_blocks(cur, split)
        P, R = pmgr.build_transfers(blocks, split, spec, cfg.ideal_size_cap)
        f_relax = pmgr._build_f_relax(blocks[0], spec, cfg)
        smoother = pmgr._build_global_smoother(cur, lay, spec, cfg)
        coarse = pmgr.build_coarse(cur, lay, split, blocks, P, R, spec)
        levs.append(pmgr._MgrLevel(cur, lay, split, blocks, P, R, f_relax, smoother, spec))
        lay = FieldLayout(lay.field_of[split.c_rows()], lay.entity_of[split.c_rows()])
        cur = coarse
    term = amg_setup(cur, cfg.amg_terminal)
    return pmgr.MgrHierarchy(levs, cur, "amg", term, max(1, cfg.terminal_cycles), cfg.f_relax_position)


def config_from_options(opts):
    """Reference MgrConfig for problems.solver_options (two/one flow fields)."""
    levels = tuple(pmgr.MgrLevelSpec({Field(t) for t in lv["f"]}, {Field(t) for t in lv["c"]},
                                     **{k: v for k, v in lv.items() if k not in ("f", "c")})
                   for lv in opts["levels"]) if len(opts["levels"]) < 3 else ()
    return pmgr.MgrConfig(levels=levels, terminal_cycles=opts["terminal_cycles"],
                          f_relax_position=opts["f_relax_position"], npartitions=opts["npartitions"],
                          amg_f_relax=AmgConfig(**opts["amg_f_relax"]), amg_terminal=AmgConfig(**opts["amg_terminal"]))


def dump_amg(d, prefix, h, full):
    d[prefix + "sizes"] = np.array(h.level_sizes())
    for i, lv in enumerate(h.levels):
        k = f"{prefix}L{i}_"
        if full:
            d[k + "isc"] = lv.split.is_c
            put_csr(d, k + "P", lv.P)
            put_csr(d, k + "A", lv.A)
            d[k + "dtilde"] = lv.dtilde
        else:
            d[k + "isc_sha"] = hashlib.sha256(lv.split.is_c.tobytes()).hexdigest()
            d[k + "P_sha"] = dcsr(lv.P)
            d[k + "A_sha"] = dcsr(lv.A)
            d[k + "dtilde_sha"] = hashlib.sha256((lv.dtilde + 0.0).tobytes()).hexdigest()
    if full:
        put_csr(d, prefix + "coarse", h.coarse_A)
    else:
        d[prefix + "coarse_sha"] = dcsr(h.coarse_A)


# option variants of the reference API exercised on a small two-phase problem
VARIANTS = {
    "v1": dict(levels=(dict(f={Field.U}, c={Field.S, Field.P}, f_relax="amg", f_relax_sweeps=2,
                            interp="injection_only", n_max=4),
                       dict(f={Field.S}, c={Field.P}, f_relax="jacobi")),
               cfg=dict(terminal_cycles=1, f_relax_position="pre")),
    "v3": dict(levels=(dict(f={Field.U}, c={Field.S, Field.P}, f_relax="amg", n_max=4),
                       dict(f={Field.S}, c={Field.P}, f_relax="none")),
               cfg=dict(terminal_cycles=1, f_relax_position="pre")),
    "v2": dict(levels=(dict(f={Field.U}, c={Field.S, Field.P}, f_relax="amg"),
                       dict(f={Field.S}, c={Field.P}, f_relax="jacobi", f_relax_sweeps=2)),
               cfg=dict(terminal_cycles=2, f_relax_position="post")),
    # hybrid l1-GS (the reference's default smoother semantics) with 16 partitions
    "v4": dict(levels=(dict(f={Field.U}, c={Field.S, Field.P}, f_relax="amg", n_max=4),
                       dict(f={Field.S}, c={Field.P}, f_relax="jacobi")),
               cfg=dict(terminal_cycles=1, f_relax_position="pre"), f_parts=16, t_parts=16),
    # level-2 global smoothers of default_three_level (mgr.py:104-120)
    "v5": dict(levels=(dict(f={Field.U}, c={Field.S, Field.P}, f_relax="amg", n_max=4),
                       dict(f={Field.S}, c={Field.P}, f_relax="jacobi", global_smoother="ilu", ilu_fill=1)),
               cfg=dict(terminal_cycles=1, f_relax_position="pre", npartitions=1)),
    "v6": dict(levels=(dict(f={Field.U}, c={Field.S, Field.P}, f_relax="amg", n_max=4),
                       dict(f={Field.S}, c={Field.P}, f_relax="jacobi", global_smoother="ilu", ilu_fill=1)),
               cfg=dict(terminal_cycles=1, f_relax_position="pre", npartitions=8)),
    "v7": dict(levels=(dict(f={Field.U}, c={Field.S, Field.P}, f_relax="amg", n_max=4),
                       dict(f={Field.S}, c={Field.P}, f_relax="jacobi", global_smoother="hbgs", hbgs_sweeps=3)),
               cfg=dict(terminal_cycles=1, f_relax_position="pre", npartitions=1), interleaved=True),
    "v8": dict(levels=(dict(f={Field.U}, c={Field.S, Field.P}, f_relax="amg", n_max=4),
                       dict(f={Field.S}, c={Field.P}, f_relax="jacobi", global_smoother="hbgs", hbgs_sweeps=3)),
               cfg=dict(terminal_cycles=1, f_relax_position="pre", npartitions=4), interleaved=True),
    "v9": dict(levels=(dict(f={Field.U}, c={Field.S, Field.P}, f_relax="amg", n_max=4),
                       dict(f={Field.S}, c={Field.P}, f_relax="jacobi", global_smoother="ilu", ilu_fill=0)),
               cfg=dict(terminal_cycles=1, f_relax_position="pre", npartitions=3)),
}


def dump_problem(tag, pb, n_max, full, restart=100, four_field=False, variant=None, opts=None, max_iters=1000):
    A = CsrMatrix(pb.n, pb.n, pb.row_offsets, pb.col_indices, pb.values)
    lay = FieldLayout(pb.field_of, pb.entity_of)
    if opts is not None:  # problems.solver_options (the production configurations)
        cfg = config_from_options(opts)
        restart, max_iters = opts["restart"], opts["max_iters"]
        h = setup_4field(A, lay, None, cfg, opts) if four_field else pmgr.mgr_setup(A, lay, cfg)
    elif variant is not None:
        V = VARIANTS[variant]
        if V.get("interleaved"):
            lay = FieldLayout(pb.field_of, pb.entity_of, psp.Ordering.FLOW_INTERLEAVED)
        levels = tuple(pmgr.MgrLevelSpec(lv["f"], lv["c"], **{k: x for k, x in lv.items() if k not in ("f", "c")})
                       for lv in V["levels"])
        base = parity_config(levels, V.get("f_parts", JACOBI), V.get("t_parts", JACOBI))
        cfg = pmgr.MgrConfig(levels=levels, amg_f_relax=base.amg_f_relax, amg_terminal=base.amg_terminal,
                             **V["cfg"])
        h = pmgr.mgr_setup(A, lay, cfg)
    elif four_field:
        cfg = parity_config(())
        h = setup_4field(A, lay, n_max, cfg)
    else:
        cfg = parity_config(levels_for(pb, n_max))
        h = pmgr.mgr_setup(A, lay, cfg)
    d = {}
    d["input_sha"] = np.array(digest(pb.row_offsets, pb.col_indices, pb.values))
    d["rhs_sha"] = np.array(hashlib.sha256(pb.rhs.tobytes()).hexdigest())
    d["mgr_sizes"] = np.array(h.level_sizes())
    for i, lv in enumerate(h.levels):
        k = f"mgr{i}_"
        nxt = h.levels[i + 1].A if i + 1 < len(h.levels) else h.terminal_A
        if full:
            d[k + "isc"] = lv.split.is_c
            put_csr(d, k + "P", lv.P)
            put_csr(d, k + "coarse", nxt)
        else:
            d[k + "isc_sha"] = hashlib.sha256(lv.split.is_c.tobytes()).hexdigest()
            d[k + "P_sha"] = dcsr(lv.P)
            d[k + "coarse_sha"] = dcsr(nxt)
        if isinstance(lv.f_relax, pmgr._AmgFRelax):
            dump_amg(d, k + "amg_", lv.f_relax.hierarchy, full)
        if isinstance(lv.global_smoother, pmgr._IluGlobal):
            put_csr(d, k + "ilu", lv.global_smoother.factors.lu)
            d[k + "ilu_dpos"] = lv.global_smoother.factors.diag_pos
        if lv.global_smoother is not None:
            rng_s = np.random.default_rng(99)
            vs = rng_s.standard_normal(lv.A.nrows)
            d[k + "gs_v"] = vs
            d[k + "gs_z"] = lv.global_smoother.apply(vs)
    dump_amg(d, "term_", h.terminal_solver, full)
    rng = np.random.default_rng(1234)
    v = rng.standard_normal(pb.n)
    d["apply_v"] = v
    d["apply_z"] = pmgr.mgr_apply(h, v)
    x, st = gmres(lambda y: matvec(A, y), h.apply, pb.rhs,
                  cfg=GmresConfig(restart=restart, max_iters=max_iters, rtol=1e-6))
    d["gmres_iters"] = np.array(st.iterations)
    d["gmres_hist"] = st.residual_history
    d["gmres_x"] = x
    d["gmres_conv"] = np.array(st.converged)
    d["versions"] = np.array(json.dumps(VERSIONS))
    path = os.path.join(OUT, f"ref_{tag}.npz")
    np.savez_compressed(path, **d)
    print(tag, pb.n, pb.nnz, "levels", h.level_sizes(), "its", st.iterations, "->", path,
          os.path.getsize(path) // 1024, "KiB")


def dump_units():
    """Kernel-level cases on the reference's own fixture shapes."""
    sys.path.insert(0, os.path.join(os.path.dirname(REF), "tests"))
    from common import diag_dominant_random, laplacian_2d

    d = {}
    rng = np.random.default_rng(7)
    # spgemm (structural) / subtract / sparsify on random two-field matrices
    for t in range(6):
        A = diag_dominant_random(rng, 40, density=0.15)
        B = diag_dominant_random(rng, 40, density=0.15)
        put_csr(d, f"u{t}_A", A)
        put_csr(d, f"u{t}_B", B)
        put_csr(d, f"u{t}_AB", spgemm(A, B))
        put_csr(d, f"u{t}_AmB", subtract(A, B))
        ent = np.repeat(np.arange(20, dtype=np.int32), 2)
        lay = FieldLayout(np.tile([1, 2], 20).astype(np.int8), ent)
        d[f"u{t}_ent"] = ent
        for nm in (0, 2, 4):
            put_csr(d, f"u{t}_sp{nm}", sparsify(A, lay, nm))
        # Galerkin product with scipy semantics, as amg.py:200-202
        sA, sB = A.to_scipy(), B.to_scipy()
        put_csr(d, f"u{t}_gal", CsrMatrix.from_scipy((sB.T @ sA @ sB).tocsr()))
        # hybrid l1-GS sweeps with 1, 3 and n partitions
        b = rng.standard_normal(40)
        x = rng.standard_normal(40)
        d[f"u{t}_b"] = b
        d[f"u{t}_x"] = x
        for npart in (1, 3, JACOBI):
            parts = PartitionSet.contiguous(40, npart)
            dt = l1_diagonal(A, parts)
            d[f"u{t}_dt{min(npart, 99)}"] = dt
            d[f"u{t}_gsf{min(npart, 99)}"] = l1_gs_sweep(A, b, x, "forward", parts, dt)
            d[f"u{t}_gsb{min(npart, 99)}"] = l1_gs_sweep(A, b, x, "backward", parts, dt)
    # AMG on anisotropic 2-D Laplacians (test_amg.py's fixture family)
    for t, (nx, eps) in enumerate(((12, 1.0), (16, 0.01), (20, 1.0))):
        L = laplacian_2d(nx, eps_y=eps)
        put_csr(d, f"lap{t}_A", L)
        S = strength_graph(L, 0.25)
        put_csr(d, f"lap{t}_S", S)
        for npart in (1, JACOBI):
            h = amg_setup(L, AmgConfig(npartitions=npart))
            tag = f"lap{t}_p{min(npart, 99)}_"
            dump_amg(d, tag, h, True)
            b = np.random.default_rng(t).standard_normal(L.nrows)
            d[tag + "b"] = b
            d[tag + "vcyc"] = amg_vcycle(h, b, np.zeros(L.nrows))
            x, st = gmres(lambda y: matvec(L, y), lambda y: amg_vcycle(h, y, np.zeros(L.nrows)), b,
                          cfg=GmresConfig(restart=30, max_iters=200, rtol=1e-8))
            d[tag + "its"] = np.array(st.iterations)
            d[tag + "hist"] = st.residual_history
            d[tag + "x"] = x
    d["versions"] = np.array(json.dumps(VERSIONS))
    path = os.path.join(OUT, "ref_units.npz")
    np.savez_compressed(path, **d)
    print("units ->", path, os.path.getsize(path) // 1024, "KiB")


def main():
    os.makedirs(OUT, exist_ok=True)
    which = sys.argv[1:] or ["units", "c1_6", "c2_6", "c4_4", "c1_16", "c2_32"]
    if "units" in which:
        dump_units()
    if "c1_6" in which:
        dump_problem("c1_6", problems.make_c1(seed=3, n=6), None, True)
    if "c2_6" in which:
        dump_problem("c2_6", problems.make_c2(seed=5, n=6), 4, True)
    if "c4_4" in which:
        dump_problem("c4_4", problems.make_c4(seed=9, n=4), 4, True, four_field=True)
    if "c1_16" in which:
        dump_problem("c1_16", problems.make_c1(seed=0, n=16), None, False)
    if "c2_32" in which:
        dump_problem("c2_32", problems.make_c2(seed=0, n=32), 4, False)
    if "c4_16" in which:
        dump_problem("c4_16", problems.make_c4(seed=0, n=16), 4, False, four_field=True)
    if "c2_6_v1" in which:
        dump_problem("c2_6_v1", problems.make_c2(seed=5, n=6), None, True, variant="v1")
    if "c2_6_v2" in which:
        dump_problem("c2_6_v2", problems.make_c2(seed=5, n=6), None, True, variant="v2")
    if "c2_6_v3" in which:
        dump_problem("c2_6_v3", problems.make_c2(seed=5, n=6), None, True, variant="v3")
    for v in ("v4", "v5", "v6", "v7", "v8", "v9"):
        if f"c2_6_{v}" in which:
            dump_problem(f"c2_6_{v}", problems.make_c2(seed=5, n=6), None, True, variant=v)
    if "c3_16" in which:
        dump_problem("c3_16", problems.make_c3(seed=0, n=16), 4, False, restart=100)
    # the production configurations (problems.solver_options) at 32^3
    if "c3_32p" in which:
        pb = problems.make_c3(seed=0, n=32)
        dump_problem("c3_32p", pb, None, False, opts=problems.solver_options("C3", pb))
    if "c4_32p" in which:
        pb = problems.make_c4(seed=0, n=32)
        dump_problem("c4_32p", pb, None, False, four_field=True, opts=problems.solver_options("C4", pb))
    # parity configuration at 32^3: the iteration counts the GPU must reproduce
    # (C3 stalls into 2801 iterations -- the algorithm, not the device)
    if "c4_32" in which:
        dump_problem("c4_32", problems.make_c4(seed=0, n=32), 4, False, four_field=True)
    if "c3_32" in which:
        dump_problem("c3_32", problems.make_c3(seed=0, n=32), 4, False, max_iters=3000)


if __name__ == "__main__":
    main()
