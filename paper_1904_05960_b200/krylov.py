"""Right-preconditioned restarted GMRES: the reference `poromgr.krylov`
surface (krylov.py:15-125).

Fast path: when `apply_A` is a matrix (CsrMatrix / DeviceCsr /
`sparse.operator(A)`) and `apply_M_inv` is None, an MgrHierarchy or its bound
`.apply`, the whole solve runs inside libpmgr.so (`pmgr_gmres`, or
`pmgr_gmres_host` when b is a NumPy array).

Generic path: arbitrary callables (e.g. `lambda v: matvec(A, v)`) are
called on float64 CUDA tensors; the Arnoldi projections use libpmgr's
multi-dot / multi-axpy kernels and the tiny Hessenberg algebra stays on the
host exactly as in the reference.  Either way the vectors never leave the GPU.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .mgr import MgrHierarchy
from .sparse import (CsrMatrix, DeviceCsr, MatvecOperator, as_device_csr, current_stream, empty_device,
                     is_device_tensor, ptr, to_device)

__all__ = ["GmresConfig", "SolveStats", "gmres"]


@dataclass(frozen=True)
class GmresConfig:
    restart: int = 50
    max_iters: int = 500
    rtol: float = 1e-6
    atol: float = 1e-12

    def __post_init__(self):
        if self.restart < 1:
            raise ValueError("restart must be >= 1")
        if self.rtol <= 0 or self.atol <= 0:
            raise ValueError("tolerances must be positive")


@dataclass
class SolveStats:
    iterations: int
    residual_history: np.ndarray
    converged: bool


def _as_matrix(op):
    if isinstance(op, (CsrMatrix, DeviceCsr)):
        return as_device_csr(op)
    if isinstance(op, MatvecOperator):
        return op.dev
    return None


def _as_mgr(op):
    if op is None:
        return None, True
    if isinstance(op, MgrHierarchy):
        return op, True
    if getattr(op, "__func__", None) is MgrHierarchy.apply and isinstance(getattr(op, "__self__", None),
                                                                           MgrHierarchy):
        return op.__self__, True
    return None, False


def gmres(apply_A, apply_M_inv, b, x0=None, cfg: GmresConfig = GmresConfig()):
    """Solve A x = b with right preconditioning M^-1; returns (x, SolveStats).

    Convergence when ||b - A x|| <= max(rtol * ||b - A x0||, atol); an
    Arnoldi breakdown counts as convergence in the generated subspace.
    """
    A = _as_matrix(apply_A)
    M, m_ok = _as_mgr(apply_M_inv)
    if A is not None and m_ok:
        return _gmres_native(A, M, b, x0, cfg)
    if A is not None:
        apply_A = MatvecOperator(A)
    return _gmres_generic(apply_A, apply_M_inv, b, x0, cfg)


def _gmres_native(A: DeviceCsr, M, b, x0, cfg):
    n = A.nrows
    c = _lib.GmresCfg(int(cfg.restart), int(cfg.max_iters), float(cfg.rtol), float(cfg.atol))
    st = _lib.GmresStats()
    cap = int(cfg.max_iters) + 2
    hist = np.zeros(cap)
    L = _lib.lib()
    mh = M.handle if M is not None else None
    if is_device_tensor(b):
        bd = to_device(b, n)
        x = to_device(x0, n).clone() if x0 is not None else empty_device(n).zero_()
        nz = 1 if x0 is not None and bool((x != 0).any()) else 0
        _lib.check(L.pmgr_gmres(A.handle, mh, ptr(bd), ptr(x), nz, ctypes.byref(c), ctypes.byref(st),
                                hist.ctypes.data, cap, current_stream()))
    else:
        bh = np.ascontiguousarray(b, dtype=np.float64)
        if len(bh) != n:
            raise ValueError("b does not match the operator")
        if x0 is None:  # the library zeroes x on the device and writes every entry back
            x = np.empty(n)
            nz = 0
        else:
            x = np.array(x0, dtype=np.float64, copy=True)
            nz = 1 if np.any(x) else 0
        _lib.check(L.pmgr_gmres_host(A.handle, mh, bh.ctypes.data, x.ctypes.data, nz, ctypes.byref(c),
                                     ctypes.byref(st), hist.ctypes.data, cap, current_stream()))
    return x, SolveStats(int(st.iterations), hist[:st.history_len].copy(), bool(st.converged))


def _call(op, v):
    out = op(v)
    if not is_device_tensor(out):
        out = to_device(out)
    return out


class DeviceVectors:
    """Vector algebra of the generic GMRES loop on libpmgr kernels (the
    reference's numpy algebra in krylov.py:52-117): norms, CGS2 projections,
    basis combinations and axpby all run in libpmgr.so on the current stream;
    only the (j+1) projection coefficients and the norms reach the host, where
    the Hessenberg/Givens algebra lives exactly as in the reference."""

    def __init__(self):
        self.L = _lib.lib()
        self.s = current_stream()

    def zeros(self, shape):
        import torch

        return torch.zeros(shape, dtype=torch.float64, device="cuda")

    def norm(self, v) -> float:
        out = ctypes.c_double()
        _lib.check(self.L.pmgr_vec_norm2(ptr(v), v.numel(), ctypes.byref(out), self.s))
        return out.value

    def axpby(self, a, x, b, y):
        """y = a x + b y in place (b = 0 ignores y's contents); returns y."""
        _lib.check(self.L.pmgr_vec_axpby(float(a), ptr(x), float(b), ptr(y), y.numel(), self.s))
        return y

    def project(self, V, k, w):
        """CGS2: w -= V[:k]^T (V[:k] w), twice; returns the summed coefficients."""
        h = np.zeros(k)
        hd = self.zeros(k)
        n = w.numel()
        for _ in range(2):
            _lib.check(self.L.pmgr_multidot(ptr(V), n, k, ptr(w), ptr(hd), self.s))
            _lib.check(self.L.pmgr_multiaxpy(ptr(V), n, k, ptr(hd), ptr(w), self.s))
            h += hd.cpu().numpy()
        return h

    def combine(self, V, j, y):
        """u = sum_{k<j} y_k V_k."""
        yd = to_device(np.ascontiguousarray(y, dtype=np.float64))
        n = V.shape[1]
        u = self.zeros(n)
        _lib.check(self.L.pmgr_combine(ptr(V), n, n, j, ptr(yd), ptr(u), self.s))
        return u


def gmres_loop(vec, apply_A, apply_M, b, x, nonzero_x0, restart, max_iters, rtol, atol):
    """Restarted right-preconditioned GMRES (reference krylov.py:39-117) over
    an abstract vector algebra `vec` (DeviceVectors here; dist.DistVectors for
    row-distributed slices).  Returns (x, iterations, history, converged)."""
    from scipy.linalg import solve_triangular

    M = (lambda v: v) if apply_M is None else apply_M
    n = b.numel()
    r = vec.axpby(1.0, b, -1.0, apply_A(x).clone()) if nonzero_x0 else b.clone()
    beta = vec.norm(r)
    hist = [beta]
    tol = max(rtol * beta, atol)
    total = 0
    m = restart
    brk = False
    while beta > tol and total < max_iters:
        V = vec.zeros((m + 1, n))
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        vec.axpby(1.0 / beta, r, 0.0, V[0])
        g[0] = beta
        j = 0
        while j < m and total < max_iters:
            w = apply_A(M(V[j])).contiguous()
            if w.untyped_storage().data_ptr() == V.untyped_storage().data_ptr():
                w = w.clone()  # an identity operator hands back the basis row itself
            H[:j + 1, j] = vec.project(V, j + 1, w)
            hn = vec.norm(w)
            H[j + 1, j] = hn
            if hn > 1e-12 * max(float(np.linalg.norm(H[:j + 2, j])), 1e-300):
                vec.axpby(1.0 / hn, w, 0.0, V[j + 1])
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
            cs[j], sn[j] = H[j, j] / rho, H[j + 1, j] / rho
            H[j, j], H[j + 1, j] = rho, 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            total += 1
            j += 1
            hist.append(abs(float(g[j])))
            if abs(g[j]) <= tol or brk:
                break
        if j > 0:
            y = solve_triangular(H[:j, :j], g[:j], lower=False)
            x = vec.axpby(1.0, M(vec.combine(V, j, y)), 1.0, x.clone())
            r = vec.axpby(1.0, b, -1.0, apply_A(x).clone())
            beta = vec.norm(r)
            hist[-1] = beta
        if brk:
            break
    return x, total, np.array(hist), bool(beta <= tol)


def _gmres_generic(apply_A, apply_M_inv, b, x0, cfg):
    """Reference krylov.py:39-117 over device vectors and arbitrary callables.

    The Krylov vectors live on the device.  Callables see what the caller's
    b is: float64 CUDA tensors when b is one, NumPy arrays when b is a NumPy
    array (the reference's contract: `lambda v: lu @ v` keeps working; each
    call then copies v to the host and the result back)."""
    host_in = not is_device_tensor(b)
    bd = to_device(b)
    n = bd.numel()
    vec = DeviceVectors()
    x = vec.zeros(n) if x0 is None else to_device(x0, n).clone()
    nonzero = x0 is not None and bool((x != 0).any())

    def wrap(op):
        if op is None:
            return None
        if host_in:
            return lambda v: _call(op, v.cpu().numpy())
        return lambda v: _call(op, v)

    x, total, hist, conv = gmres_loop(vec, wrap(apply_A), wrap(apply_M_inv), bd, x, nonzero, cfg.restart,
                                      cfg.max_iters, cfg.rtol, cfg.atol)
    out = x.cpu().numpy() if host_in else x
    return out, SolveStats(total, hist, conv)
