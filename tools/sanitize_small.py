"""Small driver for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
every kernel family once on C1 and a reduced C2/C4, both Bi-CGSTAB schedules, both
GMRES orthogonalisations, CSR and SELL, one- and two-sided scaling.  Checks the
results against the oracle so a silent corruption also fails."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_0812_2769_b200 as gsk  # noqa: E402
import workloads  # noqa: E402

for name, N in (("C1", None), ("C2", 40), ("C4", 12)):
    s = workloads.generate(name, N=N)
    A = gsk.CSR.from_system(s)
    As, bs, d = gsk.gs_scale(A, s["b"], 2)
    vo, bo, _ = oracle.gs_scale(s["row_ptr"], s["val"], s["b"], 2)
    assert np.array_equal(As.val.cpu().numpy(), vo)
    A2, b2, sv = gsk.gs_scale_sym(A, s["b"], 2)
    for fmt in ("csr", "sell"):
        for sched in ("split", "fused"):
            P = gsk.Plan(As, fmt=fmt, schedule=sched)
            x, h, r = P.bicgstab(bs, tol=1e-8, maxit=60)
            xo, ho, ro = oracle.bicgstab(s["row_ptr"], s["col"], vo, bo, 1e-8, 60)
            assert np.array_equal(h, ho), (name, fmt, sched)
            P.close()
        for orth in ("mgs", "cgs2"):
            P = gsk.Plan(As, fmt=fmt, orth=orth)
            x, h, r = P.gmres(bs, m=8, tol=1e-8, maxit=20)
            xo, ho, ro = oracle.gmres(s["row_ptr"], s["col"], vo, bo, 8, 1e-8, 20, orth=orth)
            assert np.array_equal(h, ho), (name, fmt, orth)
            y = P.spmv(bs)
            P.close()
    print(name, "ok", flush=True)
print("sanitize driver done")
