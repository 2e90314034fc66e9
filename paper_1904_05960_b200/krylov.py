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


def _gmres_generic(apply_A, apply_M_inv, b, x0, cfg):
    """Reference krylov.py:39-117 over device vectors and arbitrary callables."""
    import torch
    from scipy.linalg import solve_triangular

    host_in = not is_device_tensor(b)
    bd = to_device(b)
    n = bd.numel()
    x = torch.zeros(n, dtype=torch.float64, device="cuda") if x0 is None else to_device(x0, n).clone()
    M = (lambda v: v) if apply_M_inv is None else apply_M_inv
    L = _lib.lib()
    s = current_stream()
    r = bd - _call(apply_A, x) if bool((x != 0).any()) else bd.clone()
    beta = float(torch.linalg.vector_norm(r))
    hist = [beta]
    tol = max(cfg.rtol * beta, cfg.atol)
    total = 0
    m = cfg.restart
    if beta > tol:
        while total < cfg.max_iters:
            V = torch.zeros((m + 1, n), dtype=torch.float64, device="cuda")
            H = np.zeros((m + 1, m))
            cs = np.zeros(m)
            sn = np.zeros(m)
            g = np.zeros(m + 1)
            V[0] = r / beta
            g[0] = beta
            j = 0
            brk = False
            hd = torch.zeros(m + 1, dtype=torch.float64, device="cuda")
            while j < m and total < cfg.max_iters:
                w = _call(apply_A, _call(M, V[j])).contiguous()
                # CGS2 projections on the device
                h = np.zeros(j + 1)
                for _ in range(2):
                    _lib.check(L.pmgr_multidot(ptr(V), n, j + 1, ptr(w), ptr(hd), s))
                    _lib.check(L.pmgr_multiaxpy(ptr(V), n, j + 1, ptr(hd), ptr(w), s))
                    h += hd[:j + 1].cpu().numpy()
                H[:j + 1, j] = h
                hn = float(torch.linalg.vector_norm(w))
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
                u = torch.from_numpy(y).cuda() @ V[:j]
                x = x + _call(M, u)
                r = bd - _call(apply_A, x)
                beta = float(torch.linalg.vector_norm(r))
                hist[-1] = beta
            if beta <= tol or brk:
                break
    out = x.cpu().numpy() if host_in else x
    return out, SolveStats(total, np.array(hist), bool(beta <= tol))
