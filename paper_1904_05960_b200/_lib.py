"""ctypes binding of libpmgr.so (include/pmgr.h) and error mapping.

The CUDA library is the only compute path: if it is missing, every call
raises instead of falling back to anything on the CPU.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PMGR_LIB") or os.path.join(_HERE, "libpmgr.so")  # PMGR_LIB: A/B tooling only

c_i8p = ctypes.POINTER(ctypes.c_int8)
c_i32p = ctypes.POINTER(ctypes.c_int32)
c_i64p = ctypes.POINTER(ctypes.c_int64)
c_dp = ctypes.POINTER(ctypes.c_double)
vp = ctypes.c_void_p

PMGR_OK = 0
PMGR_ERR_INVALID = 1
PMGR_ERR_SINGULAR_DIAG = 2
PMGR_ERR_L1_VANISHES = 3
PMGR_ERR_DENSE_CAP = 4
PMGR_ERR_CUDA = 5
PMGR_ERR_NOT_SUPPORTED = 6
PMGR_ERR_OOM = 7
PMGR_ERR_INTERP_DIAG = 8
PMGR_ERR_FIELDS = 9
PMGR_ERR_ZERO_PIVOT = 10

INTERP = {"injection_only": 0, "injection_jacobi": 1, "ideal": 2}
RESTRICT = {"injection": 0, "jacobi": 1, "ideal": 2}
FRELAX = {"none": 0, "jacobi": 1, "amg": 2, "exact": 3}
SMOOTHER = {"none": 0, "hbgs": 1, "ilu": 2}


class AmgCfg(ctypes.Structure):
    _fields_ = [("strength_threshold", ctypes.c_double), ("max_levels", ctypes.c_int32),
                ("coarse_size_cutoff", ctypes.c_int32), ("num_functions", ctypes.c_int32),
                ("cycles", ctypes.c_int32), ("npartitions", ctypes.c_int64)]


class LevelSpec(ctypes.Structure):
    _fields_ = [("f_mask", ctypes.c_uint64), ("c_mask", ctypes.c_uint64), ("interp", ctypes.c_int32),
                ("restrict_", ctypes.c_int32), ("f_relax", ctypes.c_int32), ("f_relax_sweeps", ctypes.c_int32),
                ("global_smoother", ctypes.c_int32), ("n_max", ctypes.c_int32), ("quasi_impes", ctypes.c_int32),
                ("amg_num_functions", ctypes.c_int32), ("ilu_fill", ctypes.c_int32), ("hbgs_sweeps", ctypes.c_int32)]


class MgrCfg(ctypes.Structure):
    _fields_ = [("terminal_cycles", ctypes.c_int32), ("f_relax_post", ctypes.c_int32),
                ("amg_f_relax", AmgCfg), ("amg_terminal", AmgCfg), ("npartitions", ctypes.c_int64),
                ("flow_interleaved", ctypes.c_int32)]


class GmresCfg(ctypes.Structure):
    _fields_ = [("restart", ctypes.c_int32), ("max_iters", ctypes.c_int32), ("rtol", ctypes.c_double),
                ("atol", ctypes.c_double)]


ALLTOALLV_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p),
                                ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_void_p),
                                ctypes.POINTER(ctypes.c_int64))
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_int64)


class NcclId(ctypes.Structure):
    _fields_ = [("internal", ctypes.c_char * 128)]


class Assembly(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32), ("phases", ctypes.c_int32),
                ("h", ctypes.c_double), ("V", ctypes.c_double), ("phi", ctypes.c_double), ("ct", ctypes.c_double),
                ("dt", ctypes.c_double), ("biot", ctypes.c_double), ("mu", ctypes.c_double * 3)] + \
               [(nm, ctypes.c_void_p) for nm in ("E", "kx", "ky", "kz", "sats", "pstate", "K0", "bvec")]


class GmresStats(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("converged", ctypes.c_int32), ("history_len", ctypes.c_int32),
                ("restarts", ctypes.c_int32)]


# name -> (restype, argtypes); mirrors include/pmgr.h one to one
SIGNATURES = {
    "pmgr_version": (ctypes.c_int, []),
    "pmgr_last_error": (ctypes.c_char_p, []),
    "pmgr_last_error_index": (ctypes.c_int64, []),
    "pmgr_launch_count": (ctypes.c_int64, []),
    "pmgr_release_cached_memory": (ctypes.c_int, []),
    "pmgr_csr_create": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, vp, vp, vp, ctypes.c_int,
                                       ctypes.c_int, vp, ctypes.POINTER(vp)]),
    "pmgr_csr_destroy": (ctypes.c_int, [vp]),
    "pmgr_csr_info": (ctypes.c_int, [vp, c_i64p, c_i64p, c_i64p]),
    "pmgr_csr_download": (ctypes.c_int, [vp, vp, vp, vp, ctypes.c_int, vp]),
    "pmgr_spmv": (ctypes.c_int, [vp, vp, vp, vp]),
    "pmgr_csr_permute": (ctypes.c_int, [vp, vp, vp, ctypes.POINTER(vp)]),
    "pmgr_amg_setup": (ctypes.c_int, [vp, ctypes.POINTER(AmgCfg), vp, ctypes.POINTER(vp)]),
    "pmgr_amg_destroy": (ctypes.c_int, [vp]),
    "pmgr_amg_num_levels": (ctypes.c_int, [vp, c_i32p]),
    "pmgr_amg_level_sizes": (ctypes.c_int, [vp, c_i64p]),
    "pmgr_amg_flagged_rows": (ctypes.c_int, [vp, c_i64p]),
    "pmgr_amg_vcycle": (ctypes.c_int, [vp, vp, vp, vp, vp]),
    "pmgr_amg_export_csr": (ctypes.c_int, [vp, ctypes.c_int32, ctypes.c_int32, vp, ctypes.POINTER(vp)]),
    "pmgr_amg_export_vec": (ctypes.c_int, [vp, ctypes.c_int32, ctypes.c_int32, vp, vp]),
    "pmgr_mgr_setup": (ctypes.c_int, [vp, vp, vp, ctypes.POINTER(LevelSpec), ctypes.c_int32,
                                      ctypes.POINTER(MgrCfg), vp, ctypes.POINTER(vp)]),
    "pmgr_mgr_destroy": (ctypes.c_int, [vp]),
    "pmgr_mgr_num_levels": (ctypes.c_int, [vp, c_i32p]),
    "pmgr_mgr_level_sizes": (ctypes.c_int, [vp, c_i64p]),
    "pmgr_mgr_apply_bytes": (ctypes.c_int, [vp, vp, vp]),
    "pmgr_mgr_apply": (ctypes.c_int, [vp, vp, vp, vp]),
    "pmgr_mgr_export_csr": (ctypes.c_int, [vp, ctypes.c_int32, ctypes.c_int32, vp, ctypes.POINTER(vp)]),
    "pmgr_mgr_export_vec": (ctypes.c_int, [vp, ctypes.c_int32, ctypes.c_int32, vp, vp]),
    "pmgr_mgr_amg": (ctypes.c_int, [vp, ctypes.c_int32, ctypes.POINTER(vp)]),
    "pmgr_gmres": (ctypes.c_int, [vp, vp, vp, vp, ctypes.c_int, ctypes.POINTER(GmresCfg),
                                  ctypes.POINTER(GmresStats), vp, ctypes.c_int32, vp]),
    "pmgr_gmres_host": (ctypes.c_int, [vp, vp, vp, vp, ctypes.c_int, ctypes.POINTER(GmresCfg),
                                       ctypes.POINTER(GmresStats), vp, ctypes.c_int32, vp]),
    "pmgr_prof_enable": (ctypes.c_int, [ctypes.c_int]),
    "pmgr_prof_query": (ctypes.c_int, [ctypes.c_int32, c_i64p, c_dp, c_dp]),
    "pmgr_multidot": (ctypes.c_int, [vp, ctypes.c_int64, ctypes.c_int32, vp, vp, vp]),
    "pmgr_multiaxpy": (ctypes.c_int, [vp, ctypes.c_int64, ctypes.c_int32, vp, vp, vp]),
    "pmgr_vec_norm2": (ctypes.c_int, [vp, ctypes.c_int64, vp, vp]),
    "pmgr_vec_axpby": (ctypes.c_int, [ctypes.c_double, vp, ctypes.c_double, vp, ctypes.c_int64, vp]),
    "pmgr_combine": (ctypes.c_int, [vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, vp, vp, vp]),
    "pmgr_nccl_get_id": (ctypes.c_int, [ctypes.POINTER(NcclId)]),
    "pmgr_transport_host_create": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, vp, vp, vp, vp]),
    "pmgr_transport_nccl_create": (ctypes.c_int, [ctypes.POINTER(NcclId), ctypes.c_int32, ctypes.c_int32,
                                                  ctypes.POINTER(vp)]),
    "pmgr_transport_destroy": (ctypes.c_int, [vp]),
    "pmgr_dist_create": (ctypes.c_int, [vp, vp, vp, ctypes.c_int32, ctypes.c_int32, vp, vp, ctypes.POINTER(vp)]),
    "pmgr_dist_info": (ctypes.c_int, [vp, c_i64p, c_i64p]),
    "pmgr_dist_apply": (ctypes.c_int, [vp, vp, vp, vp]),
    "pmgr_dist_spmv": (ctypes.c_int, [vp, vp, vp, vp]),
    "pmgr_dist_gmres": (ctypes.c_int, [vp, vp, vp, ctypes.c_int, ctypes.POINTER(GmresCfg),
                                       ctypes.POINTER(GmresStats), vp, ctypes.c_int32, vp]),
    "pmgr_dist_destroy": (ctypes.c_int, [vp]),
    "pmgr_assemble_poromech": (ctypes.c_int, [ctypes.POINTER(Assembly), vp, ctypes.POINTER(vp)]),
    "pmgr_dist_emulate": (ctypes.c_int, [vp, vp, vp, ctypes.c_int32, ctypes.c_int32, vp, vp,
                                         ctypes.POINTER(GmresCfg), ctypes.POINTER(GmresStats), vp]),
    "pmgr_csr_rows": (ctypes.c_int, [vp, ctypes.c_int64, ctypes.c_int64, vp, ctypes.POINTER(vp)]),
    "pmgr_dist_setup": (ctypes.c_int, [vp, vp, vp, vp, ctypes.c_int32, ctypes.POINTER(MgrCfg), vp, ctypes.c_int32,
                                       ctypes.c_int32, vp, vp, ctypes.POINTER(vp)]),
    "pmgr_dist_setup_emulate": (ctypes.c_int, [vp, vp, vp, vp, ctypes.c_int32, ctypes.POINTER(MgrCfg), vp,
                                               ctypes.c_int32, ctypes.c_int32, vp, vp, ctypes.POINTER(GmresCfg),
                                               ctypes.POINTER(GmresStats), vp]),
}

_lib = None


class LibraryMissing(RuntimeError):
    pass


def lib():
    """Load libpmgr.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(f"{LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; "
                                 "g.build()'` (there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class ZeroPivotError(ArithmeticError):
    def __init__(self, row: int):
        self.row = int(row)
        super().__init__(f"zero pivot at row {int(row)}")


def check(status: int):
    """Turn a pmgr_status into the reference's exception type."""
    if status == PMGR_OK:
        return
    L = lib()
    msg = L.pmgr_last_error().decode(errors="replace")
    if status in (PMGR_ERR_INVALID, PMGR_ERR_SINGULAR_DIAG, PMGR_ERR_L1_VANISHES, PMGR_ERR_INTERP_DIAG,
                  PMGR_ERR_FIELDS):
        raise ValueError(msg)
    if status == PMGR_ERR_NOT_SUPPORTED:
        raise NotImplementedError(msg)
    if status == PMGR_ERR_ZERO_PIVOT:
        raise ZeroPivotError(int(L.pmgr_last_error_index()))
    if status == PMGR_ERR_OOM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def launch_count() -> int:
    return int(lib().pmgr_launch_count())


def release_cached_memory() -> None:
    """Return the device blocks libpmgr keeps for reuse (memory of destroyed
    matrices and hierarchies) to the CUDA driver."""
    check(lib().pmgr_release_cached_memory())
