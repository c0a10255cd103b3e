"""Row-class applicability and solve time per scaling variant (argv: config, default C4)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0812_2769_b200 as gsk  # noqa: E402
import workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
s = workloads.generate(name)
A0 = gsk.CSR.from_system(s)
b0 = torch.tensor(s["b"], device="cuda")
_, _, d2 = gsk.gs_scale(A0, b0, 2)
for label, p in (("none", None), ("GS1", 1), ("GS2", 2), ("sym", "sym")):
    A = gsk.CSR(A0.row_ptr, A0.col, A0.val.clone())
    b = b0.clone()
    w = d2
    if p == "sym":
        A, b, w = gsk.gs_scale_sym(A, b, 2)
    elif p is not None:
        A, b, dp = gsk.gs_scale(A, b, p, inplace=True)
        w = None if p == 2 else d2 / dp
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    P = gsk.Plan(A, fmt="sell", weights=w, sell_index="classes")
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    _, _, r = P.bicgstab(b, tol=1e-8, maxit=300, hist=False)
    print(label, "classes", P.num_classes(), "slots", P.num_slots(), "plan_ms", round((t1 - t0) * 1e3, 1),
          "ms/it", round(r["solve_ms"] / max(r["iterations"], 1), 4), flush=True)
    P.close()
