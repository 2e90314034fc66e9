"""B200-native MGR-preconditioned GMRES (arxiv/paper_1904_05960 hot path).

Drop-in for the reference package `poromgr`'s solver surface:

    from paper_1904_05960_b200 import sparse, amg, mgr, krylov
    h = mgr.mgr_setup(A, layout, cfg)
    x, stats = krylov.gmres(A, h.apply, b, cfg=krylov.GmresConfig(restart=100))

All compute runs in libpmgr.so (hand-written sm_100a CUDA, C ABI in
include/pmgr.h); torch only supplies device buffers and the current stream.
"""

from . import problems  # noqa: F401  (host-side input generator)

__all__ = ["sparse", "amg", "mgr", "krylov", "problems"]


def __getattr__(name):
    if name in ("sparse", "amg", "mgr", "krylov"):
        import importlib

        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
