"""One on-chip Bi-CGSTAB and one GMRES(20) solve of C1 after GS(2) (ncu target for the
small.cu kernels):  ncu -k regex:small_ --launch-skip 2 -c 2 python tools/prof_small.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0812_2769_b200 as gsk  # noqa: E402
import workloads  # noqa: E402

s = workloads.generate("C1")
A, b, _ = gsk.gs_scale(gsk.CSR.from_system(s), s["b"], 2)
P = gsk.Plan(A)
for _ in range(2):
    x, h, r = P.bicgstab(b, tol=1e-8, maxit=2000)
    print("bicgstab", r["iterations"], r["solve_ms"])
    x, h, r = P.gmres(b, m=20, tol=1e-8, maxit=2000)
    print("gmres", r["iterations"], r["solve_ms"])
