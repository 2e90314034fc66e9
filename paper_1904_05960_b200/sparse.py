"""Sparse core: the reference `poromgr.sparse` surface, device-backed.

Host containers (`CsrMatrix`, `FieldLayout`, `CfSplitting`, `Field`,
`Ordering`) keep the reference's dtypes, invariants and error messages
(reference sparse.py:42-253) so existing callers keep working.  Compute
(`matvec`) runs in libpmgr.so on the GPU; a matrix is uploaded once and the
device copy is cached on the (immutable) host object.

Vectors may be NumPy arrays (copied to and from the device per call, like
the reference's pure functions) or float64 CUDA torch tensors (stay on the
device; torch only provides the buffer and the current stream).
"""

from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _lib

__all__ = ["Field", "Ordering", "CsrMatrix", "DeviceCsr", "FieldLayout", "CfSplitting", "matvec",
           "operator", "MatvecOperator", "field_from_name"]


class Field(enum.IntEnum):
    """Physical field tag of a degree of freedom (reference sparse.py:42-47).

    S2 (= 3) extends the reference enum for the three-phase configuration
    (second saturation), which the reference cannot express.
    """

    U = 0
    S = 1
    P = 2
    S2 = 3


_FIELD_BY_NAME = {"u": Field.U, "s": Field.S, "p": Field.P, "s2": Field.S2}


def field_from_name(name: str) -> Field:
    try:
        return _FIELD_BY_NAME[name.lower()]
    except KeyError:
        raise ValueError(f"unknown field tag {name!r}, expected one of u/s/p") from None


class Ordering(enum.Enum):
    FIELD_BLOCKED = "field_blocked"
    FLOW_INTERLEAVED = "flow_interleaved"


# ---------------------------------------------------------------------------
# device plumbing (torch is used for buffers and the current stream only)
# ---------------------------------------------------------------------------


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device visible: libpmgr runs on the GPU only (no CPU fallback)")
    return torch


def current_stream():
    return ctypes.c_void_p(_torch().cuda.current_stream().cuda_stream)


def is_device_tensor(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor) and x.is_cuda


def to_device(x, n=None):
    """float64 contiguous CUDA tensor view of x (copy only when needed)."""
    torch = _torch()
    if isinstance(x, torch.Tensor):
        t = x
        if not t.is_cuda:
            t = t.cuda()
        if t.dtype != torch.float64:
            t = t.to(torch.float64)
        t = t.contiguous()
    else:
        t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()
    if n is not None and t.numel() != n:
        raise ValueError(f"vector has length {t.numel()}, expected {n}")
    return t


def empty_device(n):
    torch = _torch()
    return torch.empty(int(n), dtype=torch.float64, device="cuda")


def ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def back_like(t, like):
    """Return t in the container type of `like` (numpy in -> numpy out)."""
    if is_device_tensor(like):
        return t
    _torch().cuda.current_stream().synchronize()
    return t.cpu().numpy()


# ---------------------------------------------------------------------------
# CSR
# ---------------------------------------------------------------------------


class DeviceCsr:
    """A CSR matrix resident in libpmgr-owned device memory (pmgr_csr)."""

    def __init__(self, handle, nrows, ncols, nnz):
        self._h = ctypes.c_void_p(handle) if not isinstance(handle, ctypes.c_void_p) else handle
        self.nrows, self.ncols, self.nnz = int(nrows), int(ncols), int(nnz)

    @classmethod
    def from_arrays(cls, nrows, ncols, row_offsets, col_indices, values, validate=True) -> "DeviceCsr":
        """Upload from NumPy arrays or CUDA tensors (int64 / int32 / float64)."""
        L = _lib.lib()
        on_dev = is_device_tensor(values)
        if on_dev:
            torch = _torch()
            ro = row_offsets.to(torch.int64).contiguous()
            ci = col_indices.to(torch.int32).contiguous()
            va = values.to(torch.float64).contiguous()
            p = [ptr(ro), ptr(ci), ptr(va)]
            keep = (ro, ci, va)
        else:
            ro = np.ascontiguousarray(row_offsets, dtype=np.int64)
            ci = np.ascontiguousarray(col_indices, dtype=np.int32)
            va = np.ascontiguousarray(values, dtype=np.float64)
            p = [ctypes.c_void_p(a.ctypes.data) for a in (ro, ci, va)]
            keep = (ro, ci, va)
        nnz = len(va)
        out = ctypes.c_void_p()
        _lib.check(L.pmgr_csr_create(nrows, ncols, nnz, p[0], p[1], p[2], 1 if on_dev else 0,
                                     1 if validate else 0, current_stream(), ctypes.byref(out)))
        del keep
        return cls(out, nrows, ncols, nnz)

    @property
    def handle(self):
        return self._h

    @property
    def shape(self):
        return (self.nrows, self.ncols)

    def download(self):
        """(row_offsets, col_indices, values) host copies, unvalidated."""
        ro = np.empty(self.nrows + 1, dtype=np.int64)
        ci = np.empty(self.nnz, dtype=np.int32)
        va = np.empty(self.nnz, dtype=np.float64)
        _lib.check(_lib.lib().pmgr_csr_download(self._h, ro.ctypes.data, ci.ctypes.data, va.ctypes.data, 0,
                                                current_stream()))
        return ro, ci, va

    def to_host(self) -> "CsrMatrix":
        ro = np.empty(self.nrows + 1, dtype=np.int64)
        ci = np.empty(self.nnz, dtype=np.int32)
        va = np.empty(self.nnz, dtype=np.float64)
        _lib.check(_lib.lib().pmgr_csr_download(self._h, ro.ctypes.data, ci.ctypes.data, va.ctypes.data, 0,
                                                current_stream()))
        return CsrMatrix(self.nrows, self.ncols, ro, ci, va)

    def __matmul__(self, x):
        return matvec(self, x)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None and _lib._lib is not None:
            _lib._lib.pmgr_csr_destroy(h)
            self._h = None


@dataclass(frozen=True)
class CsrMatrix:
    """Compressed sparse row matrix with canonical structure (reference
    sparse.py:65-165): int64 offsets, int32 strictly increasing columns per
    row, float64 values; explicit zeros are legal."""

    nrows: int
    ncols: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "row_offsets", np.ascontiguousarray(self.row_offsets, dtype=np.int64))
        object.__setattr__(self, "col_indices", np.ascontiguousarray(self.col_indices, dtype=np.int32))
        object.__setattr__(self, "values", np.ascontiguousarray(self.values, dtype=np.float64))
        # the matrix is immutable (reference sparse.py:1-7) and its device copy
        # is a snapshot taken on first use: expose read-only views so an in-place
        # update (A.values[:] = ...) fails instead of leaving a stale device copy
        for name in ("row_offsets", "col_indices", "values"):
            v = getattr(self, name).view()
            v.flags.writeable = False
            object.__setattr__(self, name, v)
        self._validate()

    def _validate(self):
        ro, ci = self.row_offsets, self.col_indices
        if ro.shape != (self.nrows + 1,):
            raise ValueError(f"row_offsets has length {ro.shape[0]}, expected nrows+1={self.nrows + 1}")
        if ro[0] != 0 or ro[-1] != len(ci) or len(ci) != len(self.values):
            raise ValueError("row_offsets endpoints inconsistent with nnz")
        if np.any(ro[1:] < ro[:-1]):
            raise ValueError("row_offsets must be non-decreasing")
        if len(ci):
            if ci.min() < 0 or ci.max() >= self.ncols:
                raise ValueError("column index out of range")
            steps = np.diff(ci.astype(np.int64))
            bad = np.flatnonzero(steps <= 0) + 1
            if len(bad):
                starts = np.zeros(len(ci), dtype=bool)
                starts[ro[:-1][ro[:-1] < len(ci)]] = True
                if not np.all(starts[bad]):
                    raise ValueError("column indices must be strictly increasing within each row")

    # -- constructors (host side, as the reference) ----------------------

    @classmethod
    def from_scipy(cls, m) -> "CsrMatrix":
        m = m.tocsr()
        if not m.has_sorted_indices:
            m = m.copy()
            m.sort_indices()
        return cls(m.shape[0], m.shape[1], m.indptr, m.indices, m.data)

    @classmethod
    def from_dense(cls, a, keep_zeros: bool = False) -> "CsrMatrix":
        a = np.asarray(a, dtype=np.float64)
        nr, nc = a.shape
        if keep_zeros:
            return cls(nr, nc, np.arange(nr + 1, dtype=np.int64) * nc, np.tile(np.arange(nc, dtype=np.int32), nr),
                       a.ravel())
        mask = a != 0.0
        ro = np.concatenate([[0], np.cumsum(mask.sum(axis=1))])
        rows, cols = np.nonzero(mask)
        return cls(nr, nc, ro, cols, a[rows, cols])

    @classmethod
    def from_coo(cls, nrows, ncols, rows, cols, vals) -> "CsrMatrix":
        """Build from COO triplets; duplicates are summed."""
        import scipy.sparse as sp

        m = sp.coo_matrix((vals, (rows, cols)), shape=(nrows, ncols)).tocsr()
        m.sort_indices()
        return cls(nrows, ncols, m.indptr, m.indices, m.data)

    @classmethod
    def identity(cls, n: int) -> "CsrMatrix":
        return cls(n, n, np.arange(n + 1), np.arange(n), np.ones(n))

    # -- views ------------------------------------------------------------

    @property
    def nnz(self) -> int:
        return len(self.values)

    @property
    def shape(self) -> tuple:
        return (self.nrows, self.ncols)

    def to_scipy(self):
        import scipy.sparse as sp

        m = sp.csr_matrix((self.values, self.col_indices, self.row_offsets), shape=self.shape, copy=False)
        m.has_sorted_indices = True
        return m

    def to_dense(self) -> np.ndarray:
        out = np.zeros(self.shape)
        rows = np.repeat(np.arange(self.nrows), np.diff(self.row_offsets))
        out[rows, self.col_indices] = self.values
        return out

    def diagonal(self) -> np.ndarray:
        n = min(self.nrows, self.ncols)
        rows = np.repeat(np.arange(self.nrows), np.diff(self.row_offsets))
        d = np.zeros(n)
        hit = (rows == self.col_indices) & (rows < n)
        d[rows[hit]] = self.values[hit]
        return d

    def transpose(self) -> "CsrMatrix":
        return CsrMatrix.from_scipy(self.to_scipy().T.tocsr())

    def row_pattern(self, i: int) -> np.ndarray:
        return self.col_indices[self.row_offsets[i]:self.row_offsets[i + 1]]

    # -- device ------------------------------------------------------------

    def device(self) -> DeviceCsr:
        """The cached device copy (uploaded on first use)."""
        d = self.__dict__.get("_dev")
        if d is None:
            d = DeviceCsr.from_arrays(self.nrows, self.ncols, self.row_offsets, self.col_indices, self.values,
                                      validate=False)
            object.__setattr__(self, "_dev", d)
        return d


def as_device_csr(A) -> DeviceCsr:
    if isinstance(A, DeviceCsr):
        return A
    if isinstance(A, CsrMatrix):
        return A.device()
    raise TypeError(f"expected CsrMatrix or DeviceCsr, got {type(A).__name__}")


@dataclass(frozen=True)
class FieldLayout:
    """dof -> (field, entity) map (reference sparse.py:167-216)."""

    field_of: np.ndarray
    entity_of: np.ndarray
    ordering: Ordering = Ordering.FIELD_BLOCKED

    def __post_init__(self):
        object.__setattr__(self, "field_of", np.ascontiguousarray(self.field_of, dtype=np.int8))
        object.__setattr__(self, "entity_of", np.ascontiguousarray(self.entity_of, dtype=np.int32))
        if self.field_of.shape != self.entity_of.shape:
            raise ValueError("field_of and entity_of must have equal length")
        if self.ordering == Ordering.FLOW_INTERLEAVED:
            s = np.flatnonzero(self.field_of == Field.S)
            p = np.flatnonzero(self.field_of == Field.P)
            if len(s) != len(p):
                raise ValueError("interleaved layout requires one S and one P dof per cell")
            if len(s):
                s = s[np.argsort(self.entity_of[s], kind="stable")]
                p = p[np.argsort(self.entity_of[p], kind="stable")]
                if np.any(np.abs(s - p) != 1):
                    raise ValueError("interleaved layout requires adjacent S/P dofs per cell")

    @property
    def ndofs(self) -> int:
        return len(self.field_of)

    def fields_present(self) -> set:
        return {Field(v) for v in np.unique(self.field_of)}

    def dofs_of(self, f: Field) -> np.ndarray:
        return np.flatnonzero(self.field_of == f)

    def restrict(self, idx: np.ndarray) -> "FieldLayout":
        """Layout of the kept dofs.  Unlike the reference (mgr.py:359 x
        sparse.py:180-189), a restriction that no longer pairs S/P
        dofs falls back to FIELD_BLOCKED instead of raising."""
        fo, eo = self.field_of[idx], self.entity_of[idx]
        try:
            return FieldLayout(fo, eo, self.ordering)
        except ValueError:
            return FieldLayout(fo, eo, Ordering.FIELD_BLOCKED)

    @classmethod
    def single_field(cls, n: int, f: Field = Field.P) -> "FieldLayout":
        return cls(np.full(n, int(f), dtype=np.int8), np.arange(n, dtype=np.int32))

    @classmethod
    def interleaved_flow(cls, ncells: int) -> "FieldLayout":
        f = np.empty(2 * ncells, dtype=np.int8)
        f[0::2] = Field.S
        f[1::2] = Field.P
        e = np.repeat(np.arange(ncells, dtype=np.int32), 2)
        return cls(f, e, Ordering.FLOW_INTERLEAVED)


@dataclass(frozen=True)
class CfSplitting:
    """Disjoint C/F partition of matrix rows, order preserving (reference
    sparse.py:219-253)."""

    is_c: np.ndarray
    c_index: np.ndarray = field(default=None)
    f_index: np.ndarray = field(default=None)

    def __post_init__(self):
        object.__setattr__(self, "is_c", np.ascontiguousarray(self.is_c, dtype=bool))
        if self.c_index is None:
            ci = np.full(len(self.is_c), -1, dtype=np.int64)
            ci[self.is_c] = np.arange(int(self.is_c.sum()))
            fi = np.full(len(self.is_c), -1, dtype=np.int64)
            fi[~self.is_c] = np.arange(int((~self.is_c).sum()))
            object.__setattr__(self, "c_index", ci)
            object.__setattr__(self, "f_index", fi)

    @property
    def n(self) -> int:
        return len(self.is_c)

    @property
    def n_c(self) -> int:
        return int(self.is_c.sum())

    @property
    def n_f(self) -> int:
        return self.n - self.n_c

    def c_rows(self) -> np.ndarray:
        return np.flatnonzero(self.is_c)

    def f_rows(self) -> np.ndarray:
        return np.flatnonzero(~self.is_c)


# ---------------------------------------------------------------------------
# kernels
# ---------------------------------------------------------------------------


def matvec(A, x):
    """y = A x on the device (reference sparse.py:261-266)."""
    dA = as_device_csr(A)
    n = x.numel() if is_device_tensor(x) else len(x)
    if n != dA.ncols:
        raise ValueError(f"matvec dimension mismatch: A is {dA.nrows}x{dA.ncols}, x has length {n}")
    xd = to_device(x)
    y = empty_device(dA.nrows)
    _lib.check(_lib.lib().pmgr_spmv(dA.handle, ptr(xd), ptr(y), current_stream()))
    return back_like(y, x)


class MatvecOperator:
    """Callable v -> A v that gmres() recognises and runs fully on device."""

    def __init__(self, A):
        self.A = A
        self.dev = as_device_csr(A)

    def __call__(self, v):
        return matvec(self.dev, v)

    @property
    def shape(self):
        return self.dev.shape


def operator(A) -> MatvecOperator:
    return MatvecOperator(A)


# ---------------------------------------------------------------------------
# Matrix Market IO (reference sparse.py:484-502: general real coordinate
# format, 1-based on disk, 17 significant digits so values round-trip)
# ---------------------------------------------------------------------------


def write_matrix_market(path, A: CsrMatrix) -> None:
    from scipy.io import mmwrite

    mmwrite(str(path), A.to_scipy().tocoo(), precision=17, symmetry="general")


def read_matrix_market(path) -> CsrMatrix:
    import scipy.sparse as sp
    from scipy.io import mmread

    m = mmread(str(path), spmatrix=False) if "spmatrix" in mmread.__code__.co_varnames else mmread(str(path))
    if not sp.issparse(m):
        raise ValueError(f"{path}: not a coordinate-format matrix")
    return CsrMatrix.from_scipy(sp.csr_matrix(m))


def write_vector(path, v) -> None:
    from scipy.io import mmwrite

    mmwrite(str(path), np.asarray(v, dtype=np.float64).reshape(-1, 1), precision=17)


def read_vector(path) -> np.ndarray:
    from scipy.io import mmread

    return np.asarray(mmread(str(path)), dtype=np.float64).ravel()
