"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the MGR-GMRES hot path.

A restatement of the reference package `poromgr` (arxiv/paper_1904_05960,
/root/reference/pkg/src/poromgr) on top of the C kernels in oracle.c.  Only
tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may import
this module; the product (paper_1904_05960_b200/) never does.

Parity configuration: the AMG smoother is exercised with the
reference's own contiguous-partition semantics, so `npartitions >= n` gives
l1-Jacobi (bitwise equal to the reference's hybrid l1-GS with one row per
partition) and `npartitions = 1` gives sequential l1-GS.

Pinned: tests/test_oracle_golden.py checks this module bitwise (patterns and
setup values) and to 1e-12 (applies, GMRES) against tests/golden/*.npz, which
oracle/make_golden.py produced by running the reference itself.
"""

from __future__ import annotations

import ctypes
import logging
import os
from dataclasses import dataclass, field

import numpy as np

logger = logging.getLogger(__name__)

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

DENSE_SOLVE_CAP = 20000  # reference amg.py:32


def build(force: bool = False) -> str:
    """Compile oracle.c (gcc, no FMA contraction) into oracle/_build/."""
    import subprocess

    src = os.path.join(_HERE, "oracle.c")
    os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O3", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
                               "-shared", "-o", _LIB_PATH, src, "-lm"])
    return _LIB_PATH


class _OCsr(ctypes.Structure):
    _fields_ = [("nrows", ctypes.c_int64), ("ncols", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("ro", ctypes.POINTER(ctypes.c_int64)), ("ci", ctypes.POINTER(ctypes.c_int32)),
                ("v", ctypes.POINTER(ctypes.c_double))]


def lib():
    global _lib
    if _lib is None:
        build()  # no-op unless oracle.c is newer than the library
        _lib = ctypes.CDLL(_LIB_PATH)
        _lib.o_free.argtypes = [ctypes.c_void_p]
        for name in ("o_direct_interp", "o_l1diag", "o_lu_factor"):
            getattr(_lib, name).restype = ctypes.c_int64
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data)


# ---------------------------------------------------------------------------
# CSR container (reference CsrMatrix, sparse.py:65-165)
# ---------------------------------------------------------------------------


@dataclass
class Csr:
    nrows: int
    ncols: int
    ro: np.ndarray
    ci: np.ndarray
    v: np.ndarray

    def __post_init__(self):
        self.ro = np.ascontiguousarray(self.ro, dtype=np.int64)
        self.ci = np.ascontiguousarray(self.ci, dtype=np.int32)
        self.v = np.ascontiguousarray(self.v, dtype=np.float64)

    @property
    def nnz(self):
        return len(self.v)

    def to_struct(self):
        s = _OCsr(self.nrows, self.ncols, self.nnz,
                  self.ro.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                  self.ci.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                  self.v.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        return s

    @staticmethod
    def from_struct(s: _OCsr) -> "Csr":
        n, nnz = s.nrows, s.nnz
        ro = np.ctypeslib.as_array(s.ro, shape=(n + 1,)).copy()
        ci = np.ctypeslib.as_array(s.ci, shape=(max(nnz, 1),))[:nnz].copy()
        v = np.ctypeslib.as_array(s.v, shape=(max(nnz, 1),))[:nnz].copy()
        L = lib()
        L.o_free(ctypes.cast(s.ro, ctypes.c_void_p))
        L.o_free(ctypes.cast(s.ci, ctypes.c_void_p))
        L.o_free(ctypes.cast(s.v, ctypes.c_void_p))
        return Csr(s.nrows, s.ncols, ro, ci, v)

    def to_dense(self):
        out = np.zeros((self.nrows, self.ncols))
        rows = np.repeat(np.arange(self.nrows), np.diff(self.ro))
        out[rows, self.ci] = self.v
        return out

    def diagonal(self):
        d = np.zeros(self.nrows)
        lib().o_diagonal(ctypes.c_int64(self.nrows), _p(self.ro), _p(self.ci), _p(self.v), _p(d))
        return d

    def rows_of_entries(self):
        return np.repeat(np.arange(self.nrows, dtype=np.int64), np.diff(self.ro))


def spmv(A: Csr, x) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(A.nrows)
    lib().o_spmv(ctypes.c_int64(A.nrows), _p(A.ro), _p(A.ci), _p(A.v), _p(x), _p(y))
    return y


def transpose(A: Csr) -> Csr:
    s = A.to_struct()
    out = _OCsr()
    lib().o_transpose(ctypes.byref(s), ctypes.byref(out))
    return Csr.from_struct(out)


def spgemm(X: Csr, Y: Csr, keep_structural: bool) -> Csr:
    sx, sy, out = X.to_struct(), Y.to_struct(), _OCsr()
    lib().o_spgemm(ctypes.byref(sx), ctypes.byref(sy), ctypes.c_int(1 if keep_structural else 0),
                   ctypes.byref(out))
    return Csr.from_struct(out)


def subtract(A: Csr, B: Csr) -> Csr:
    sa, sb, out = A.to_struct(), B.to_struct(), _OCsr()
    lib().o_subtract(ctypes.byref(sa), ctypes.byref(sb), ctypes.byref(out))
    return Csr.from_struct(out)


def sparsify(M: Csr, entity_of: np.ndarray, n_max: int) -> Csr:
    ent = np.ascontiguousarray(entity_of, dtype=np.int32)
    sm, out = M.to_struct(), _OCsr()
    lib().o_sparsify(ctypes.byref(sm), _p(ent), ctypes.c_int64(n_max), ctypes.byref(out))
    return Csr.from_struct(out)


# ---------------------------------------------------------------------------
# smoothers (reference smoothers.py:41-124)
# ---------------------------------------------------------------------------


def partition_starts(n: int, nparts: int, align: int = 1) -> np.ndarray:
    """Contiguous near-equal partitions (reference smoothers.py:67-75)."""
    nparts = max(1, min(nparts, max(1, n // max(align, 1))))
    b = np.round(np.linspace(0, n, nparts + 1) / align).astype(np.int64) * align
    b[0], b[-1] = 0, n
    return np.unique(b)


def l1_diagonal(A: Csr, starts: np.ndarray) -> np.ndarray:
    d = np.empty(A.nrows)
    bad = lib().o_l1diag(ctypes.c_int64(A.nrows), _p(A.ro), _p(A.ci), _p(A.v),
                         ctypes.c_int64(len(starts) - 1), _p(starts), _p(d))
    if bad >= 0:
        raise ValueError(f"l1 diagonal vanishes at row {int(bad)}")
    return d


def l1_sweep(A: Csr, b, x, starts, dtilde, forward: bool) -> np.ndarray:
    out = np.array(x, dtype=np.float64, copy=True)
    pre = np.empty_like(out)
    b = np.ascontiguousarray(b, dtype=np.float64)
    lib().o_l1gs(ctypes.c_int64(A.nrows), _p(A.ro), _p(A.ci), _p(A.v),
                 ctypes.c_int64(len(starts) - 1), _p(starts), _p(dtilde), _p(b), _p(out), _p(pre),
                 ctypes.c_int(1 if forward else 0))
    return out


# ---------------------------------------------------------------------------
# level-2 global smoothers (reference smoothers.py:127-224, mgr.py:275-292)
# ---------------------------------------------------------------------------


class ZeroPivotError(ArithmeticError):
    def __init__(self, row: int):
        self.row = int(row)
        super().__init__(f"zero pivot at row {int(row)}")


def restrict_to_partitions(A: Csr, starts: np.ndarray) -> Csr:
    """Drop couplings crossing partition boundaries (smoothers.py:215-224)."""
    rows = A.rows_of_entries()
    part = np.searchsorted(starts, rows, side="right") - 1
    keep = (A.ci >= starts[part]) & (A.ci < starts[part + 1])
    kept = np.flatnonzero(keep)
    ro = np.concatenate([[0], np.cumsum(np.bincount(rows[kept], minlength=A.nrows))]).astype(np.int64)
    return Csr(A.nrows, A.ncols, ro, A.ci[kept], A.v[kept])


def _iluk(A: Csr, k: int):
    L = lib()
    n = A.nrows
    lptr = np.zeros(n + 1, dtype=np.int64)
    dpos = np.full(n, -1, dtype=np.int64)
    tot = ctypes.c_int64()
    L.o_iluk_symbolic.restype = ctypes.c_int64
    cnt = L.o_iluk_symbolic(ctypes.c_int64(n), _p(A.ro), _p(A.ci), ctypes.c_int(k), ctypes.c_int64(0), _p(lptr),
                            None, None, _p(dpos), ctypes.byref(tot))
    ind = np.zeros(max(cnt, 1), dtype=np.int32)
    lev = np.zeros(max(cnt, 1), dtype=np.int32)
    L.o_iluk_symbolic(ctypes.c_int64(n), _p(A.ro), _p(A.ci), ctypes.c_int(k), ctypes.c_int64(max(cnt, 1)), _p(lptr),
                      _p(ind), _p(lev), _p(dpos), None)
    data = np.zeros(max(cnt, 1))
    L.o_iluk_numeric.restype = ctypes.c_int64
    fail = L.o_iluk_numeric(ctypes.c_int64(n), _p(A.ro), _p(A.ci), _p(A.v), _p(lptr), _p(ind), _p(dpos), _p(data))
    return Csr(n, n, lptr, ind[:cnt], data[:cnt]), dpos, int(fail)


def ilu_factor(A: Csr, k: int, zero_pivot_shift=None):
    """ILU(k) without pivoting; on a zero pivot, retry once on
    A + shift*max(|diag|, 1)*I (scipy sum: exact zeros dropped) (smoothers.py:159-188)."""
    lu, dpos, fail = _iluk(A, k)
    if fail >= 0:
        if zero_pivot_shift is None:
            raise ZeroPivotError(fail)
        shift = zero_pivot_shift * max(float(np.max(np.abs(A.diagonal()))), 1.0)
        import scipy.sparse as sp
        S = sp.csr_matrix((A.v, A.ci, A.ro), shape=(A.nrows, A.ncols)) + shift * sp.identity(A.nrows, format="csr")
        S = S.tocsr()
        S.sort_indices()
        lu, dpos, fail = _iluk(Csr(S.shape[0], S.shape[1], S.indptr.astype(np.int64), S.indices.astype(np.int32),
                                   S.data.astype(np.float64)), k)
        if fail >= 0:
            raise ZeroPivotError(fail)
    return lu, dpos


def ilu_solve(lu: Csr, dpos: np.ndarray, r) -> np.ndarray:
    z = np.empty(lu.nrows)
    r = np.ascontiguousarray(r, dtype=np.float64)
    lib().o_ilu_solve(ctypes.c_int64(lu.nrows), _p(lu.ro), _p(lu.ci), _p(lu.v), _p(dpos), _p(r), _p(z))
    return z


def offpart_abs_rowsum(A: Csr, starts: np.ndarray) -> np.ndarray:
    out = np.empty(A.nrows)
    lib().o_offpart_abs(ctypes.c_int64(A.nrows), _p(A.ro), _p(A.ci), _p(A.v), ctypes.c_int64(len(starts) - 1),
                        _p(starts), _p(out))
    return out


def hbgs_sweeps(A: Csr, field_of, entity_of, b, nsweeps: int, starts: np.ndarray) -> np.ndarray:
    """Hybrid block Gauss-Seidel over per-cell 2x2 (s, p) blocks from x = 0
    (smoothers.py:127-152): S / P dofs paired by entity."""
    s = np.flatnonzero(field_of == 1)
    s = s[np.argsort(entity_of[s], kind="stable")].astype(np.int64)
    p = np.flatnonzero(field_of == 2)
    p = p[np.argsort(entity_of[p], kind="stable")].astype(np.int64)
    add = offpart_abs_rowsum(A, starts)
    x = np.zeros(A.nrows)
    pre = np.empty(A.nrows)
    b = np.ascontiguousarray(b, dtype=np.float64)
    L = lib()
    L.o_hbgs_sweep.restype = ctypes.c_int64
    for _ in range(nsweeps):
        bad = L.o_hbgs_sweep(ctypes.c_int64(A.nrows), _p(A.ro), _p(A.ci), _p(A.v), ctypes.c_int64(len(starts) - 1),
                             _p(starts), _p(add), _p(b), _p(x), _p(pre), ctypes.c_int64(len(s)), _p(s), _p(p),
                             ctypes.c_int(1))
        if bad >= 0:
            raise ValueError(f"singular 2x2 diagonal block at cell {int(entity_of[s[bad]])}")
    return x


class GlobalSmoother:
    """_IluGlobal / _HbgsGlobal (mgr.py:275-292)."""

    def __init__(self, A: Csr, field_of, entity_of, spec, npartitions: int):
        self.kind = spec.global_smoother
        self.starts = partition_starts(A.nrows, npartitions, align=2)
        if self.kind == "ilu":
            local = restrict_to_partitions(A, self.starts) if len(self.starts) > 2 else A
            self.lu, self.dpos = ilu_factor(local, spec.ilu_fill, zero_pivot_shift=1e-8)
        else:
            self.A, self.fo, self.eo, self.nsweeps = A, field_of, entity_of, spec.hbgs_sweeps

    def apply(self, v):
        if self.kind == "ilu":
            return ilu_solve(self.lu, self.dpos, v)
        return hbgs_sweeps(self.A, self.fo, self.eo, v, self.nsweeps, self.starts)


# ---------------------------------------------------------------------------
# dense LU (LAPACK getrf/getrs stand-in, values only)
# ---------------------------------------------------------------------------


def lu_factor(a: np.ndarray):
    a = np.ascontiguousarray(a, dtype=np.float64).copy()
    n = a.shape[0]
    piv = np.zeros(n, dtype=np.int64)
    lib().o_lu_factor(ctypes.c_int64(n), _p(a), _p(piv))
    return a, piv


def lu_solve(f, b) -> np.ndarray:
    a, piv = f
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.empty_like(b)
    lib().o_lu_solve(ctypes.c_int64(len(b)), _p(a), _p(piv), _p(b), _p(x))
    return x


# ---------------------------------------------------------------------------
# classical AMG (reference amg.py:35-231)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class AmgConfig:
    strength_threshold: float = 0.25
    max_levels: int = 25
    coarse_size_cutoff: int = 64
    num_functions: int = 1
    npartitions: int = 1
    cycles: int = 1


@dataclass
class AmgLevel:
    A: Csr
    P: Csr
    R: Csr          # explicit P^T
    S_mask: np.ndarray
    is_c: np.ndarray
    dtilde: np.ndarray
    starts: np.ndarray


@dataclass
class AmgHierarchy:
    levels: list
    coarse_A: Csr
    coarse_lu: tuple
    config: AmgConfig
    flagged_f_rows: int = 0

    def level_sizes(self):
        return [lv.A.nrows for lv in self.levels] + [self.coarse_A.nrows]


def strength_mask(A: Csr, theta: float, funcs: np.ndarray) -> np.ndarray:
    mask = np.empty(A.nnz, dtype=np.uint8)
    f = np.ascontiguousarray(funcs, dtype=np.int32)
    lib().o_strength(ctypes.c_int64(A.nrows), _p(A.ro), _p(A.ci), _p(A.v), _p(f),
                     ctypes.c_double(theta), _p(mask))
    return mask


def mask_to_pattern(A: Csr, mask: np.ndarray) -> Csr:
    kept = np.flatnonzero(mask)
    rows = A.rows_of_entries()
    ro = np.concatenate([[0], np.cumsum(np.bincount(rows[kept], minlength=A.nrows))])
    return Csr(A.nrows, A.ncols, ro, A.ci[kept], np.ones(len(kept)))


def greedy_mis(S: Csr) -> np.ndarray:
    status = np.empty(S.nrows, dtype=np.int8)
    lib().o_greedy_mis(ctypes.c_int64(S.nrows), _p(S.ro), _p(S.ci), _p(status))
    return status == 1


def c_index(is_c: np.ndarray) -> np.ndarray:
    ci = np.full(len(is_c), -1, dtype=np.int64)
    ci[is_c] = np.arange(int(is_c.sum()))
    return ci


def direct_interpolation(A: Csr, mask: np.ndarray, is_c: np.ndarray, funcs: np.ndarray):
    cidx = c_index(is_c)
    isc8 = np.ascontiguousarray(is_c, dtype=np.int8)
    f = np.ascontiguousarray(funcs, dtype=np.int32)
    out = _OCsr()
    flagged = lib().o_direct_interp(ctypes.c_int64(A.nrows), _p(A.ro), _p(A.ci), _p(A.v), _p(mask),
                                    _p(isc8), _p(cidx), _p(f), ctypes.c_int64(int(is_c.sum())),
                                    ctypes.byref(out))
    if flagged == -2:
        raise ValueError("direct interpolation requires nonzero diagonals")
    P = Csr.from_struct(out)
    if flagged:
        logger.warning("%d F rows have no strong C neighbor; interpolating as zero", flagged)
    return P, int(flagged)


def galerkin(P: Csr, R: Csr, A: Csr) -> Csr:
    """(P^T A) P with exact zeros dropped after each product (scipy)."""
    return spgemm(spgemm(R, A, False), P, False)


def amg_setup(A: Csr, cfg: AmgConfig) -> AmgHierarchy:
    if A.nrows != A.ncols:
        raise ValueError("amg_setup requires a square matrix")
    levels = []
    funcs = (np.arange(A.nrows, dtype=np.int32) % cfg.num_functions).astype(np.int32)
    flagged = 0
    cur = A
    while cur.nrows > cfg.coarse_size_cutoff and len(levels) < cfg.max_levels - 1:
        mask = strength_mask(cur, cfg.strength_threshold, funcs)
        S = mask_to_pattern(cur, mask)
        is_c = greedy_mis(S)
        if int(is_c.sum()) == cur.nrows:
            break
        P, nfl = direct_interpolation(cur, mask, is_c, funcs)
        flagged += nfl
        R = transpose(P)
        nxt = galerkin(P, R, cur)
        starts = partition_starts(cur.nrows, cfg.npartitions)
        dt = l1_diagonal(cur, starts)
        levels.append(AmgLevel(cur, P, R, mask, is_c, dt, starts))
        funcs = funcs[is_c]
        cur = nxt
    if cur.nrows > DENSE_SOLVE_CAP:
        raise RuntimeError(f"coarsest AMG level of size {cur.nrows} is too large for a dense solve")
    return AmgHierarchy(levels, cur, lu_factor(cur.to_dense()), cfg, flagged)


def amg_vcycle(h: AmgHierarchy, b, x) -> np.ndarray:
    return _cycle(h, 0, np.asarray(b, dtype=np.float64), np.asarray(x, dtype=np.float64))


def _cycle(h, l, b, x):
    if l == len(h.levels):
        r = b - spmv(h.coarse_A, x) if np.any(x) else b
        return x + lu_solve(h.coarse_lu, r)
    lv = h.levels[l]
    x = l1_sweep(lv.A, b, x, lv.starts, lv.dtilde, True)
    r = b - spmv(lv.A, x)
    e = _cycle(h, l + 1, spmv(lv.R, r), np.zeros(lv.P.ncols))
    x = x + spmv(lv.P, e)
    return l1_sweep(lv.A, b, x, lv.starts, lv.dtilde, False)


# ---------------------------------------------------------------------------
# MGR (reference mgr.py:53-438), field tags generalised to any int8
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class MgrLevelSpec:
    f_fields: frozenset
    c_fields: frozenset
    f_relax: str = "jacobi"         # "jacobi" | "amg" | "none"
    f_relax_sweeps: int = 1
    n_max: int | None = None
    interp: str = "injection_jacobi"  # | "injection_only" (mgr.py:151-152)
    global_smoother: str = "none"     # | "ilu" | "hbgs" (mgr.py:388-396)
    ilu_fill: int = 1
    hbgs_sweeps: int = 3


@dataclass(frozen=True)
class MgrConfig:
    levels: tuple
    terminal_cycles: int = 1
    amg_f_relax: AmgConfig = field(default_factory=lambda: AmgConfig(strength_threshold=0.5, num_functions=3))
    amg_terminal: AmgConfig = field(default_factory=lambda: AmgConfig(strength_threshold=0.25))
    f_relax_position: str = "pre"
    npartitions: int = 1              # global smoothers' partitions (mgr.py:391)


@dataclass
class MgrLevel:
    A: Csr
    field_of: np.ndarray
    entity_of: np.ndarray
    is_c: np.ndarray
    blocks: tuple
    P: Csr
    f_relax: object
    spec: MgrLevelSpec
    dinv: np.ndarray
    smoother: object = None


@dataclass
class MgrHierarchy:
    levels: list
    terminal_A: Csr
    terminal: AmgHierarchy
    terminal_cycles: int
    f_relax_position: str = "pre"

    def apply(self, v):
        return mgr_apply(self, v)

    def level_sizes(self):
        return [lv.A.nrows for lv in self.levels] + [self.terminal_A.nrows]


def config_from_options(opts: dict) -> MgrConfig:
    """Oracle MgrConfig from problems.solver_options' plain-data description
    (the same description the library's mgr.config_from_options reads)."""
    specs = tuple(MgrLevelSpec(frozenset(lv["f"]), frozenset(lv["c"]), lv.get("f_relax", "jacobi"),
                               lv.get("f_relax_sweeps", 1), lv.get("n_max"), lv.get("interp", "injection_jacobi"),
                               lv.get("global_smoother", "none"), lv.get("ilu_fill", 1), lv.get("hbgs_sweeps", 3))
                  for lv in opts["levels"])
    return MgrConfig(levels=specs, terminal_cycles=opts.get("terminal_cycles", 1),
                     amg_f_relax=AmgConfig(**opts["amg_f_relax"]), amg_terminal=AmgConfig(**opts["amg_terminal"]),
                     f_relax_position=opts.get("f_relax_position", "pre"), npartitions=opts.get("npartitions", 1))


def extract_blocks(A: Csr, is_c: np.ndarray):
    """A_FF, A_FC, A_CF, A_CC with order-preserving renumbering and explicit
    zeros kept (reference sparse.py:269-288)."""
    rows = A.rows_of_entries()
    cols = A.ci.astype(np.int64)
    new = np.empty(A.nrows, dtype=np.int64)
    nc = int(is_c.sum())
    new[is_c] = np.arange(nc)
    new[~is_c] = np.arange(A.nrows - nc)
    out = []
    for rc in (False, True):
        for cc in (False, True):
            sel = np.flatnonzero((is_c[rows] == rc) & (is_c[cols] == cc))
            nr = nc if rc else A.nrows - nc
            ncol = nc if cc else A.nrows - nc
            r = new[rows[sel]]
            ro = np.concatenate([[0], np.cumsum(np.bincount(r, minlength=nr))])
            out.append(Csr(nr, ncol, ro, new[cols[sel]], A.v[sel]))
    return tuple(out)  # ff, fc, cf, cc


def diag_inverse(A: Csr) -> np.ndarray:
    d = A.diagonal()
    bad = np.flatnonzero(d == 0.0)
    if len(bad):
        raise ValueError(f"singular diagonal: zero or missing entry at row {int(bad[0])}")
    return 1.0 / d


def build_interp(blocks, is_c: np.ndarray, dinv, interp="injection_jacobi") -> Csr:
    """P = [W_p; I] in level order, W_p = A_FC * (-dinv_F) row-scaled
    (reference mgr.py:150-176, injection_jacobi); injection_only has no W_p."""
    a_ff, a_fc, _, _ = blocks
    if interp == "injection_only":
        a_fc = Csr(a_fc.nrows, a_fc.ncols, np.zeros(a_fc.nrows + 1, dtype=np.int64), [], [])
        dinv = np.zeros(a_fc.nrows)
    n = len(is_c)
    nc = int(is_c.sum())
    f_rows = np.flatnonzero(~is_c)
    c_rows = np.flatnonzero(is_c)
    wrows = a_fc.rows_of_entries()
    wv = a_fc.v * (-dinv)[wrows]
    cnt = np.zeros(n, dtype=np.int64)
    cnt[c_rows] = 1
    cnt[f_rows] = np.diff(a_fc.ro)
    ro = np.concatenate([[0], np.cumsum(cnt)])
    ci = np.empty(ro[-1], dtype=np.int32)
    v = np.empty(ro[-1])
    ci[ro[c_rows]] = np.arange(nc)
    v[ro[c_rows]] = 1.0
    dst = np.repeat(ro[f_rows], np.diff(a_fc.ro)) + (np.arange(a_fc.nnz) - np.repeat(a_fc.ro[:-1], np.diff(a_fc.ro)))
    ci[dst] = a_fc.ci
    v[dst] = wv
    return Csr(n, nc, ro, ci, v)


def rows_of(A: Csr, rows: np.ndarray) -> Csr:
    cnt = np.diff(A.ro)[rows]
    ro = np.concatenate([[0], np.cumsum(cnt)])
    take = np.repeat(A.ro[rows] - ro[:-1], cnt) + np.arange(ro[-1])
    return Csr(len(rows), A.ncols, ro, A.ci[take], A.v[take])


def build_coarse(A: Csr, entity_c: np.ndarray, is_c: np.ndarray, blocks, P: Csr, n_max) -> Csr:
    """T = (R A) P with the structural pattern; with n_max, the non-Galerkin
    A_CC - sparsify(A_CC - T) (reference mgr.py:212-231)."""
    ra = rows_of(A, np.flatnonzero(is_c))
    ra.v = ra.v + 0.0  # R A = 1.0*a summed from 0.0: -0.0 becomes +0.0
    ra.v[ra.v == 0.0] = 0.0
    T = spgemm(ra, P, True)
    if n_max is None:
        return T
    a_cc = blocks[3]
    corr = subtract(a_cc, T)
    kept = sparsify(corr, entity_c, n_max)
    return subtract(a_cc, kept)


def mgr_setup(A: Csr, field_of: np.ndarray, entity_of: np.ndarray, cfg: MgrConfig) -> MgrHierarchy:
    cur = A
    fo = np.asarray(field_of, dtype=np.int8)
    eo = np.asarray(entity_of, dtype=np.int32)
    levels = []
    for spec in cfg.levels:
        present = set(int(t) for t in np.unique(fo))
        if set(spec.f_fields) | set(spec.c_fields) != present:
            raise ValueError("level spec fields do not cover the fields present")
        is_c = np.isin(fo, sorted(spec.c_fields))
        if is_c.all():
            break
        blocks = extract_blocks(cur, is_c)
        # diag_inverse runs for injection_jacobi interpolation and for the
        # Jacobi F-relaxation (build_transfers mgr.py:153-155, _JacobiFRelax :241)
        need = spec.interp == "injection_jacobi" or spec.f_relax == "jacobi"
        dinv = diag_inverse(blocks[0]) if need else None
        P = build_interp(blocks, is_c, dinv, spec.interp)
        if spec.f_relax == "amg":
            acfg = cfg.amg_f_relax
            nf = 3 if set(spec.f_fields) == {0} else 1
            acfg = AmgConfig(acfg.strength_threshold, acfg.max_levels, acfg.coarse_size_cutoff, nf,
                             acfg.npartitions, acfg.cycles)
            frelax = ("amg", amg_setup(blocks[0], acfg), max(1, spec.f_relax_sweeps))
        elif spec.f_relax == "jacobi":
            frelax = ("jacobi", blocks[0], max(1, spec.f_relax_sweeps))
        else:
            frelax = None
        smoother = (GlobalSmoother(cur, fo, eo, spec, cfg.npartitions) if spec.global_smoother != "none"
                    else None)
        coarse = build_coarse(cur, eo[is_c], is_c, blocks, P, spec.n_max)
        levels.append(MgrLevel(cur, fo, eo, is_c, blocks, P, frelax, spec, dinv, smoother))
        fo, eo = fo[is_c], eo[is_c]
        cur = coarse
    term = amg_setup(cur, cfg.amg_terminal)
    return MgrHierarchy(levels, cur, term, max(1, cfg.terminal_cycles), cfg.f_relax_position)


def _f_relax_apply(lv: MgrLevel, r):
    kind = lv.f_relax[0]
    if kind == "amg":
        x = np.zeros(len(r))
        for _ in range(lv.f_relax[2]):
            x = amg_vcycle(lv.f_relax[1], r, x)
        return x
    x = lv.dinv * r
    for _ in range(lv.f_relax[2] - 1):
        x = x + lv.dinv * (r - spmv(lv.f_relax[1], x))
    return x


def mgr_apply(h: MgrHierarchy, v) -> np.ndarray:
    return _apply_level(h, 0, np.asarray(v, dtype=np.float64))


def _apply_level(h, l, v):
    if l == len(h.levels):
        e = np.zeros(len(v))
        for _ in range(h.terminal_cycles):
            e = amg_vcycle(h.terminal, v, e)
        return e
    lv = h.levels[l]
    f_rows = np.flatnonzero(~lv.is_c)
    z = None
    if lv.smoother is not None:
        z = lv.smoother.apply(v)
    if h.f_relax_position == "pre" and lv.f_relax is not None:
        if z is None:
            z = np.zeros(len(v))
            r = v
        else:
            r = v - spmv(lv.A, z)
        z[f_rows] += _f_relax_apply(lv, r[f_rows])
    r = v - spmv(lv.A, z) if z is not None else v
    ec = _apply_level(h, l + 1, r[lv.is_c])
    corr = spmv(lv.P, ec)
    z = corr if z is None else z + corr
    if h.f_relax_position == "post" and lv.f_relax is not None:
        r = v - spmv(lv.A, z)
        z[f_rows] += _f_relax_apply(lv, r[f_rows])
    return z


# ---------------------------------------------------------------------------
# GMRES (reference krylov.py:39-117): MGS Arnoldi, Givens, true residual
# ---------------------------------------------------------------------------


def gmres(apply_A, apply_M_inv, b, x0=None, restart=50, max_iters=500, rtol=1e-6, atol=1e-12):
    from scipy.linalg import solve_triangular

    b = np.asarray(b, dtype=np.float64)
    n = len(b)
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64, copy=True)
    M = (lambda v: v) if apply_M_inv is None else apply_M_inv
    r = b - apply_A(x) if np.any(x) else b.copy()
    beta = float(np.linalg.norm(r))
    hist = [beta]
    tol = max(rtol * beta, atol)
    if beta <= tol:
        return x, 0, np.array(hist), True
    m = restart
    total = 0
    while total < max_iters:
        V = np.zeros((m + 1, n))
        H = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        g = np.zeros(m + 1)
        V[0] = r / beta
        g[0] = beta
        j = 0
        brk = False
        while j < m and total < max_iters:
            w = apply_A(M(V[j]))
            for i in range(j + 1):
                H[i, j] = float(V[i] @ w)
                w = w - H[i, j] * V[i]
            hn = float(np.linalg.norm(w))
            H[j + 1, j] = hn
            if hn > 1e-12 * max(float(np.linalg.norm(H[:j + 2, j])), 1e-300):
                V[j + 1] = w / hn
            else:
                brk = True
            for i in range(j):
                t = H[i, j]
                H[i, j] = cs[i] * t + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * t + cs[i] * H[i + 1, j]
            rho = float(np.hypot(H[j, j], H[j + 1, j]))
            if rho == 0.0:
                brk = True
                break
            cs[j] = H[j, j] / rho
            sn[j] = H[j + 1, j] / rho
            H[j, j] = rho
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            total += 1
            j += 1
            hist.append(abs(float(g[j])))
            if abs(g[j]) <= tol or brk:
                break
        if j > 0:
            y = solve_triangular(H[:j, :j], g[:j], lower=False)
            x = x + M(V[:j].T @ y)
            r = b - apply_A(x)
            beta = float(np.linalg.norm(r))
            hist[-1] = beta
        if beta <= tol or brk:
            break
    return x, total, np.array(hist), bool(beta <= tol)
