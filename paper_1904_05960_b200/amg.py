"""Classical AMG: the reference `poromgr.amg` surface on the device.

`amg_setup` builds the whole hierarchy in libpmgr.so (strength, parallel
lexicographic-first MIS equal to the reference's greedy MIS, direct
interpolation, Galerkin SpGEMM, l1 diagonal, dense coarsest inverse); it is
bit-exact with reference amg.py:184-211 (patterns and values).  `amg_vcycle`
runs the V(1,1) cycle of amg.py:214-231 with the fused smoother kernels.
"""

from __future__ import annotations

import ctypes
import logging
from dataclasses import dataclass

import numpy as np

from . import _lib
from .sparse import (CfSplitting, CsrMatrix, DeviceCsr, as_device_csr, back_like, current_stream, empty_device,
                     ptr, to_device)

__all__ = ["AmgConfig", "AmgHierarchy", "amg_setup", "amg_vcycle"]

logger = logging.getLogger(__name__)

_DENSE_SOLVE_CAP = 20000


@dataclass(frozen=True)
class AmgConfig:
    """Reference AmgConfig (amg.py:35-48).  npartitions >= n gives l1-Jacobi
    (the parity configuration); smaller values give the hybrid l1-GS with
    contiguous partitions, one GPU thread per partition."""

    strength_threshold: float = 0.25
    max_levels: int = 25
    coarse_size_cutoff: int = 64
    num_functions: int = 1
    npartitions: int = 1
    cycles: int = 1

    def __post_init__(self):
        if not 0.0 <= self.strength_threshold < 1.0:
            raise ValueError("strength_threshold must be in [0, 1)")
        if self.coarse_size_cutoff < 1:
            raise ValueError("coarse_size_cutoff must be >= 1")

    def to_c(self, num_functions=None) -> _lib.AmgCfg:
        return _lib.AmgCfg(float(self.strength_threshold), int(self.max_levels), int(self.coarse_size_cutoff),
                           int(num_functions if num_functions is not None else self.num_functions), int(self.cycles),
                           int(min(self.npartitions, 2 ** 62)))


@dataclass
class AmgLevelView:
    """Host copy of one level, for inspection and parity checks."""

    A: CsrMatrix
    P: CsrMatrix
    split: CfSplitting
    dtilde: np.ndarray


def _export_dev(h, level, what) -> DeviceCsr:
    out = ctypes.c_void_p()
    _lib.check(_lib.lib().pmgr_amg_export_csr(h, level, what, current_stream(), ctypes.byref(out)))
    nr, nc, nz = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _lib.check(_lib.lib().pmgr_csr_info(out, ctypes.byref(nr), ctypes.byref(nc), ctypes.byref(nz)))
    return DeviceCsr(out, nr.value, nc.value, nz.value)


def _export_csr(h, level, what) -> CsrMatrix:
    return _export_dev(h, level, what).to_host()


class AmgHierarchy:
    """Device-resident AMG hierarchy (reference AmgHierarchy, amg.py:60-69)."""

    def __init__(self, handle, config: AmgConfig, owner=None, keepalive=None):
        self._h = handle
        self.config = config
        self._owner = owner          # MGR hierarchy owning this AMG, if borrowed
        self._keepalive = keepalive  # the operator's device copy
        n = ctypes.c_int32()
        _lib.check(_lib.lib().pmgr_amg_num_levels(self._h, ctypes.byref(n)))
        self._nlev = n.value
        f = ctypes.c_int64()
        _lib.check(_lib.lib().pmgr_amg_flagged_rows(self._h, ctypes.byref(f)))
        self.flagged_f_rows = int(f.value)

    @property
    def handle(self):
        return self._h

    def level_sizes(self):
        s = np.zeros(self._nlev + 1, dtype=np.int64)
        _lib.check(_lib.lib().pmgr_amg_level_sizes(self._h, s.ctypes.data_as(_lib.c_i64p)))
        return [int(v) for v in s]

    @property
    def levels(self):
        out = []
        sizes = self.level_sizes()
        for l in range(self._nlev):
            isc = np.zeros(sizes[l], dtype=np.int8)
            dt = np.zeros(sizes[l])
            _lib.check(_lib.lib().pmgr_amg_export_vec(self._h, l, 0, isc.ctypes.data, current_stream()))
            _lib.check(_lib.lib().pmgr_amg_export_vec(self._h, l, 1, dt.ctypes.data, current_stream()))
            out.append(AmgLevelView(_export_csr(self._h, l, 0), _export_csr(self._h, l, 1),
                                    CfSplitting(isc.astype(bool)), dt))
        return out

    @property
    def coarse_A(self) -> CsrMatrix:
        return _export_csr(self._h, 0, 2)

    def export_raw(self):
        """[(A, P, is_c, dtilde) per level], coarse A as unvalidated host arrays
        ((nrows, ncols, ro, ci, v) tuples) -- bulk export for host-side tools."""
        sizes = self.level_sizes()
        out = []
        for l in range(self._nlev):
            isc = np.zeros(sizes[l], dtype=np.int8)
            dt = np.zeros(sizes[l])
            _lib.check(_lib.lib().pmgr_amg_export_vec(self._h, l, 0, isc.ctypes.data, current_stream()))
            _lib.check(_lib.lib().pmgr_amg_export_vec(self._h, l, 1, dt.ctypes.data, current_stream()))
            a, p = _export_dev(self._h, l, 0), _export_dev(self._h, l, 1)
            out.append(((a.nrows, a.ncols) + a.download(), (p.nrows, p.ncols) + p.download(), isc.astype(bool), dt))
        c = _export_dev(self._h, 0, 2)
        return out, (c.nrows, c.ncols) + c.download()

    def vcycle(self, b, x=None):
        return amg_vcycle(self, b, x)

    def __del__(self):
        if getattr(self, "_owner", None) is None and getattr(self, "_h", None) and _lib is not None and _lib._lib is not None:
            _lib._lib.pmgr_amg_destroy(self._h)
            self._h = None


def amg_setup(A, cfg: AmgConfig = AmgConfig()) -> AmgHierarchy:
    """Build strength -> coarsen -> interpolate -> Galerkin recursively on the
    device until the operator is small enough for a dense solve."""
    dA = as_device_csr(A)
    if dA.nrows != dA.ncols:
        raise ValueError("amg_setup requires a square matrix")
    c = cfg.to_c()
    out = ctypes.c_void_p()
    _lib.check(_lib.lib().pmgr_amg_setup(dA.handle, ctypes.byref(c), current_stream(), ctypes.byref(out)))
    h = AmgHierarchy(out, cfg, keepalive=dA)
    if h.flagged_f_rows:
        logger.warning("%d F rows have no strong C neighbor; interpolating as zero", h.flagged_f_rows)
    return h


def amg_vcycle(h: AmgHierarchy, b, x=None):
    """One V(1,1) cycle (reference amg.py:214-231).  x=None or an all-zero x
    uses the zero-initial-guess path."""
    n = h.level_sizes()[0]
    bd = to_device(b, n)
    xd = None
    if x is not None:
        xd = to_device(x, n)
        if not bool((xd != 0).any()):
            xd = None
    out = empty_device(n)
    _lib.check(_lib.lib().pmgr_amg_vcycle(h.handle, ptr(bd), ptr(xd) if xd is not None else None, ptr(out),
                                          current_stream()))
    return back_like(out, b)
