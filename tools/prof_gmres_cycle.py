"""One GMRES(30) cycle on C4 after GS(2) (ncu launch-list target):
ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_gmres_cycle.py cgs2"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0812_2769_b200 as gsk  # noqa: E402
import workloads  # noqa: E402

orth = sys.argv[1] if len(sys.argv) > 1 else "mgs"
s = workloads.generate("C4")
A, b, _ = gsk.gs_scale(gsk.CSR.from_system(s), s["b"], 2)
P = gsk.Plan(A, fmt="sell", orth=orth)
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    x, h, r = P.gmres(b, m=30, tol=1e-8, maxit=30)
    print(orth, r["iterations"], r["solve_ms"], f"{1e3 * r['iterations'] / r['solve_ms']:.1f} it/s")
