"""Short driver for ncu (argv: config, default C4; layout, default sell; sell_index, default plain): GS(2), SELL plan, 2 SpMVs, 2 Bi-CGSTAB iterations
(split and fused schedules), 3 GMRES(30) steps.  Not a benchmark."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0812_2769_b200 as gsk  # noqa: E402
import workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
fmt = sys.argv[2] if len(sys.argv) > 2 else "sell"  # the bench's layout on every config
sidx = sys.argv[3] if len(sys.argv) > 3 else "plain"  # "classes": the row-class dictionary
s = workloads.generate(name)
A = gsk.CSR.from_system(s)
As, bs, _ = gsk.gs_scale(A, s["b"], 2)
x = torch.tensor(workloads.uniform(s["n"], 9, 9), device="cuda")
for sched in ("split", "fused"):
    P = gsk.Plan(As, fmt=fmt, schedule=sched, poll=2, sell_index=sidx)
    P.spmv(x)
    P.bicgstab(bs, tol=1e-8, maxit=2)
    if sched == "split":
        P.gmres(bs, m=30, tol=1e-8, maxit=3)
    P.close()
torch.cuda.synchronize()
print("done")
