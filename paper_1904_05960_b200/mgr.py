"""Multigrid reduction: the reference `poromgr.mgr` surface on the device.

`mgr_setup` (reference mgr.py:329-371) validates the level specs exactly
like the reference, then builds every level in libpmgr.so: field split,
block extraction, W_p = -D_FF^-1 A_FC, structural RAP with the optional
N_max non-Galerkin dropping, AMG / Jacobi F-relaxation and the terminal AMG.
`mgr_apply` / `MgrHierarchy.apply` run the reduction cycle of mgr.py:399-438.

The level-2 global smoothers of default_three_level (ILU(k) and hybrid block
Gauss-Seidel over partitions, mgr.py:275-292) run on the device.  Options
the reference offers but no BASELINE.json config uses and the device path
does not implement (ideal transfers, exact F / terminal solves, quasi-IMPES,
Jacobi restriction) raise NotImplementedError instead of silently running
elsewhere.
"""

from __future__ import annotations

import ctypes
import logging
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .amg import AmgConfig, AmgHierarchy
from .sparse import (CfSplitting, CsrMatrix, DeviceCsr, Field, FieldLayout, Ordering, as_device_csr, back_like,
                     current_stream, empty_device, ptr, to_device)

__all__ = ["MgrLevelSpec", "MgrConfig", "MgrHierarchy", "mgr_setup", "mgr_apply"]

logger = logging.getLogger(__name__)

_INTERP_MODES = ("injection_only", "injection_jacobi", "ideal")
_RESTRICT_MODES = ("injection", "jacobi", "ideal")
_F_RELAX_MODES = ("none", "jacobi", "amg", "exact")
_GLOBAL_SMOOTHERS = ("none", "hbgs", "ilu")


@dataclass(frozen=True)
class MgrLevelSpec:
    """One reduction level (reference mgr.py:53-83)."""

    f_fields: frozenset
    c_fields: frozenset
    interp: str = "injection_jacobi"
    restrict: str = "injection"
    f_relax: str = "jacobi"
    f_relax_sweeps: int = 1
    global_smoother: str = "none"
    hbgs_sweeps: int = 3
    ilu_fill: int = 1
    n_max: int | None = None
    quasi_impes: bool = False

    def __post_init__(self):
        object.__setattr__(self, "f_fields", frozenset(Field(f) for f in self.f_fields))
        object.__setattr__(self, "c_fields", frozenset(Field(f) for f in self.c_fields))
        if self.f_fields & self.c_fields:
            raise ValueError("f_fields and c_fields must be disjoint")
        if self.interp not in _INTERP_MODES:
            raise ValueError(f"unknown interp mode {self.interp!r}")
        if self.restrict not in _RESTRICT_MODES:
            raise ValueError(f"unknown restrict mode {self.restrict!r}")
        if self.f_relax not in _F_RELAX_MODES:
            raise ValueError(f"unknown f_relax {self.f_relax!r}")
        if self.global_smoother not in _GLOBAL_SMOOTHERS:
            raise ValueError(f"unknown global smoother {self.global_smoother!r}")
        if self.n_max is not None and self.n_max < 0:
            raise ValueError("n_max must be >= 0")

    def to_c(self) -> _lib.LevelSpec:
        fm = 0
        for f in self.f_fields:
            fm |= 1 << int(f)
        cm = 0
        for f in self.c_fields:
            cm |= 1 << int(f)
        nfun = 3 if self.f_fields == {Field.U} else 1  # reference mgr.py:382-385
        return _lib.LevelSpec(fm, cm, _lib.INTERP[self.interp], _lib.RESTRICT[self.restrict],
                              _lib.FRELAX[self.f_relax], int(self.f_relax_sweeps),
                              _lib.SMOOTHER[self.global_smoother], -1 if self.n_max is None else int(self.n_max),
                              1 if self.quasi_impes else 0, nfun, int(self.ilu_fill), int(self.hbgs_sweeps))


@dataclass(frozen=True)
class MgrConfig:
    """Reference MgrConfig (mgr.py:86-123)."""

    levels: tuple
    terminal: str = "amg"
    terminal_cycles: int = 1
    amg_f_relax: AmgConfig = field(default_factory=lambda: AmgConfig(strength_threshold=0.5, num_functions=3))
    amg_terminal: AmgConfig = field(default_factory=lambda: AmgConfig(strength_threshold=0.25))
    npartitions: int = 1
    ideal_size_cap: int = 2000
    f_relax_position: str = "pre"

    def __post_init__(self):
        object.__setattr__(self, "levels", tuple(self.levels))
        if self.terminal not in ("amg", "exact"):
            raise ValueError(f"unknown terminal solver {self.terminal!r}")
        if self.f_relax_position not in ("pre", "post"):
            raise ValueError("f_relax_position must be 'pre' or 'post'")

    @classmethod
    def default_three_level(cls, n_max: int = 4, global_smoother: str = "ilu", hbgs_sweeps: int = 3,
                            ilu_fill: int = 1, quasi_impes: bool = False, npartitions: int = 1,
                            terminal_cycles: int = 1) -> "MgrConfig":
        lvl1 = MgrLevelSpec(f_fields={Field.U}, c_fields={Field.S, Field.P}, interp="injection_jacobi",
                            restrict="injection", f_relax="amg", global_smoother="none", n_max=n_max)
        lvl2 = MgrLevelSpec(f_fields={Field.S}, c_fields={Field.P}, interp="injection_jacobi",
                            restrict="injection", f_relax="jacobi", f_relax_sweeps=1,
                            global_smoother=global_smoother, hbgs_sweeps=hbgs_sweeps, ilu_fill=ilu_fill,
                            n_max=None, quasi_impes=quasi_impes)
        return cls(levels=(lvl1, lvl2), terminal="amg", terminal_cycles=terminal_cycles, npartitions=npartitions)

    def to_c(self) -> _lib.MgrCfg:
        return _lib.MgrCfg(max(1, int(self.terminal_cycles)), 1 if self.f_relax_position == "post" else 0,
                           self.amg_f_relax.to_c(), self.amg_terminal.to_c(), int(min(self.npartitions, 2 ** 62)), 0)


class MgrLevelView:
    """Host view of one reduction level with the reference `_MgrLevel`
    attributes (mgr.py:300-310): A, layout, split, blocks, P, R, f_relax,
    global_smoother, spec, plus `coarse` (the next level's operator).  Every
    matrix is exported from the device on first access (exports are snapshots;
    the device hierarchy is what apply/gmres use)."""

    def __init__(self, h: "MgrHierarchy", level: int, split: CfSplitting, layout: FieldLayout):
        self._h, self._l = h, level
        self.split = split
        self.layout = layout
        self.spec = h.specs[level] if level < len(h.specs) else None
        self._cache = {}

    def _get(self, key, fn):
        if key not in self._cache:
            self._cache[key] = fn()
        return self._cache[key]

    @property
    def A(self) -> CsrMatrix:
        if self._l == 0:
            return self._get("A", self._h._A.to_host)
        return self._get("A", lambda: self._h._export(self._l - 1, 1))

    @property
    def P(self) -> CsrMatrix:
        return self._get("P", lambda: self._h._export(self._l, 0))

    @property
    def coarse(self) -> CsrMatrix:
        return self._get("coarse", lambda: self._h._export(self._l, 1))

    @property
    def R(self) -> CsrMatrix:
        """Injection restriction [0 I] (mgr.py:179-186 with restrict='injection')."""
        def make():
            c = self.split.c_rows()
            return CsrMatrix(len(c), self.split.n, np.arange(len(c) + 1), c, np.ones(len(c)))
        return self._get("R", make)

    @property
    def blocks(self):
        """(A_FF, A_FC, A_CF, A_CC), reference sparse.py:269-288 semantics."""
        def make():
            m = self.A.to_scipy()
            f, c = self.split.f_rows(), self.split.c_rows()
            mf, mc = m[f], m[c]
            return tuple(CsrMatrix.from_scipy(x) for x in (mf[:, f], mf[:, c], mc[:, f], mc[:, c]))
        return self._get("blocks", make)

    @property
    def f_relax(self):
        spec = self.spec
        if spec is None or spec.f_relax == "none":
            return None
        if spec.f_relax == "amg":
            return _AmgFRelaxView(self._h.amg(self._l), max(1, spec.f_relax_sweeps))
        a_ff = self.blocks[0]
        return _JacobiFRelaxView(a_ff, 1.0 / a_ff.diagonal(), max(1, spec.f_relax_sweeps))

    @property
    def global_smoother(self):
        if self.spec is None or self.spec.global_smoother == "none":
            return None
        if self.spec.global_smoother == "ilu":
            return _IluView(self._h.ilu_factors(self._l))
        return _HbgsView(self.spec.hbgs_sweeps)


@dataclass
class _AmgFRelaxView:
    """Reference _AmgFRelax (mgr.py:253-262): the device AMG on A_FF."""

    hierarchy: AmgHierarchy
    ncycles: int


@dataclass
class _JacobiFRelaxView:
    """Reference _JacobiFRelax (mgr.py:239-250)."""

    a_ff: CsrMatrix
    dinv: np.ndarray
    nsweeps: int


@dataclass
class _IluView:
    """Reference _IluGlobal (mgr.py:275-282): the combined L\\U factors."""

    lu: CsrMatrix


@dataclass
class _HbgsView:
    """Reference _HbgsGlobal (mgr.py:285-292)."""

    nsweeps: int


class MgrHierarchy:
    """Device-resident reduction hierarchy (reference MgrHierarchy, mgr.py:313-326)."""

    def __init__(self, handle, A_dev: DeviceCsr, config: MgrConfig, specs, layout: FieldLayout | None = None):
        self._h = handle
        self._A = A_dev
        self.config = config
        self.specs = tuple(specs)
        n = ctypes.c_int32()
        _lib.check(_lib.lib().pmgr_mgr_num_levels(self._h, ctypes.byref(n)))
        self._nlev = n.value
        self.terminal_cycles = max(1, config.terminal_cycles)
        self.f_relax_position = config.f_relax_position
        self._layout = layout
        self._levels = None

    @property
    def handle(self):
        return self._h

    @property
    def n(self):
        return self._A.nrows

    def apply(self, v):
        return mgr_apply(self, v)

    def apply_bytes(self):
        """(algorithmic bytes, kernel launches) of one application (the
        roofline numerator of the preconditioner; pmgr_mgr_apply_bytes)."""
        b, k = ctypes.c_double(), ctypes.c_int64()
        _lib.check(_lib.lib().pmgr_mgr_apply_bytes(self._h, ctypes.byref(b), ctypes.byref(k)))
        return b.value, k.value

    def level_sizes(self):
        s = np.zeros(self._nlev + 1, dtype=np.int64)
        _lib.check(_lib.lib().pmgr_mgr_level_sizes(self._h, s.ctypes.data_as(_lib.c_i64p)))
        return [int(v) for v in s]

    def ilu_factors(self, level: int) -> CsrMatrix:
        """Combined L\\U factors of the level's ILU(k) global smoother."""
        return self._export(level, 2)

    def _export_dev(self, level, what) -> DeviceCsr:
        out = ctypes.c_void_p()
        _lib.check(_lib.lib().pmgr_mgr_export_csr(self._h, level, what, current_stream(), ctypes.byref(out)))
        nr, nc, nz = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _lib.check(_lib.lib().pmgr_csr_info(out, ctypes.byref(nr), ctypes.byref(nc), ctypes.byref(nz)))
        return DeviceCsr(out, nr.value, nc.value, nz.value)

    def _export(self, level, what) -> CsrMatrix:
        return self._export_dev(level, what).to_host()

    @property
    def levels(self):
        """Per-level views with the reference `_MgrLevel` attributes."""
        if self._levels is None:
            out = []
            sizes = self.level_sizes()
            lay = self._layout
            for l in range(self._nlev):
                isc = np.zeros(sizes[l], dtype=np.int8)
                _lib.check(_lib.lib().pmgr_mgr_export_vec(self._h, l, 0, isc.ctypes.data, current_stream()))
                split = CfSplitting(isc.astype(bool))
                out.append(MgrLevelView(self, l, split, lay))
                lay = lay.restrict(split.c_rows()) if lay is not None else None
            self._levels = out
            self._terminal_layout = lay
        return self._levels

    @property
    def terminal_A(self) -> CsrMatrix:
        """The operator the terminal AMG works on (reference mgr.py:316)."""
        if self._nlev == 0:
            return self._A.to_host()
        return self._export(self._nlev - 1, 1)

    @property
    def terminal_kind(self) -> str:
        return self.config.terminal

    def amg(self, level: int) -> AmgHierarchy | None:
        """F-relaxation AMG of `level` (-1: terminal AMG), borrowed."""
        out = ctypes.c_void_p()
        _lib.check(_lib.lib().pmgr_mgr_amg(self._h, level, ctypes.byref(out)))
        if not out.value:
            return None
        cfg = self.config.amg_terminal if level < 0 else self.config.amg_f_relax
        return AmgHierarchy(out, cfg, owner=self)

    @property
    def terminal_solver(self) -> AmgHierarchy:
        return self.amg(-1)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None and _lib._lib is not None:
            _lib._lib.pmgr_mgr_destroy(self._h)
            self._h = None


def config_from_options(opts: dict) -> MgrConfig:
    """MgrConfig from problems.solver_options' plain-data description."""
    levels = tuple(MgrLevelSpec({Field(t) for t in lv["f"]}, {Field(t) for t in lv["c"]},
                                **{k: v for k, v in lv.items() if k not in ("f", "c")}) for lv in opts["levels"])
    return MgrConfig(levels=levels, terminal_cycles=opts.get("terminal_cycles", 1),
                     f_relax_position=opts.get("f_relax_position", "pre"), npartitions=opts.get("npartitions", 1),
                     amg_f_relax=AmgConfig(**opts["amg_f_relax"]), amg_terminal=AmgConfig(**opts["amg_terminal"]))


def mgr_setup(A, layout: FieldLayout, config: MgrConfig) -> MgrHierarchy:
    """Build the reduction hierarchy for operator A laid out by `layout`."""
    dA = as_device_csr(A)
    specs, cfg, fo0, eo0 = setup_args(dA, layout, config)
    out = ctypes.c_void_p()
    _lib.check(_lib.lib().pmgr_mgr_setup(dA.handle, fo0.ctypes.data, eo0.ctypes.data, specs, len(config.levels),
                                         ctypes.byref(cfg), current_stream(), ctypes.byref(out)))
    return MgrHierarchy(out, dA, config, config.levels, layout)


def setup_args(dA, layout: FieldLayout, config: MgrConfig):
    """Validate (mgr.py:337-352) and marshal the setup arguments of the C ABI:
    level specs, configuration, field / entity tags."""
    if dA.nrows != dA.ncols:
        raise ValueError("mgr_setup requires a square matrix")
    if layout.ndofs != dA.nrows:
        raise ValueError("layout does not match the matrix")
    if config.terminal != "amg":
        raise NotImplementedError("the exact terminal solve is not on the device path (terminal='amg')")
    # level validation mirrors mgr.py:337-352 on the host layout
    fo = layout.field_of
    for spec in config.levels:
        present = {Field(v) for v in np.unique(fo)}
        if spec.f_fields | spec.c_fields != present:
            raise ValueError(
                f"level spec fields {sorted(f.name for f in spec.f_fields | spec.c_fields)} "
                f"do not cover the fields present {sorted(f.name for f in present)}")
        if not spec.c_fields:
            raise ValueError("empty C set: nothing to reduce onto")
        is_c = np.isin(fo, [int(f) for f in spec.c_fields])
        if is_c.all():
            if len(present) != 1:
                raise ValueError("an all-C level requires a single remaining field")
            logger.info("all-C level: skipping reduction, solving directly with AMG")
            break
        fo = fo[is_c]
    if len(set(np.unique(fo).tolist())) > 1:
        logger.warning("terminal MGR grid carries %d fields; AMG works best on a single elliptic field",
                       len(set(np.unique(fo).tolist())))
    specs = (_lib.LevelSpec * max(1, len(config.levels)))(*[s.to_c() for s in config.levels])
    cfg = config.to_c()
    cfg.flow_interleaved = 1 if layout.ordering == Ordering.FLOW_INTERLEAVED else 0
    fo0 = np.ascontiguousarray(layout.field_of, dtype=np.int8)
    eo0 = np.ascontiguousarray(layout.entity_of, dtype=np.int32)
    return specs, cfg, fo0, eo0


def mgr_apply(h: MgrHierarchy, v):
    """z = M^-1 v (reference mgr.py:399-429)."""
    vd = to_device(v, h.n)
    z = empty_device(h.n)
    _lib.check(_lib.lib().pmgr_mgr_apply(h.handle, ptr(vd), ptr(z), current_stream()))
    return back_like(z, v)
