"""paper_0812_2769_b200 — geometric scaling GS(p) + Bi-CGSTAB / GMRES(m) on one B200.

Gordon & Gordon, "Geometric scaling: a simple preconditioner for certain linear
systems with discontinuous coefficients" (arXiv 0812.2769).  The hot path runs in
hand-written sm_100a kernels behind the C-ABI of ``libgsk.so`` (include/gsk.h);
this package is the thin ctypes binding (argument marshalling only).
"""
from ._gsk import (CSR, NcclComm, Plan, ShardedPlan, GskError, STATUS, SYMBOLS, LIB_PATH,  # noqa: F401
                   bicgstab_solve, dot, gmres_solve, gs_scale, gs_scale_sym, gs_unscale, launch_count, load,
                   shard_halo, shard_rows, spmv)

__all__ = ["CSR", "NcclComm", "Plan", "ShardedPlan", "GskError", "STATUS", "SYMBOLS", "LIB_PATH",
           "bicgstab_solve", "dot", "gmres_solve", "gs_scale", "gs_scale_sym", "gs_unscale", "launch_count", "load",
           "shard_halo", "shard_rows", "spmv"]
