"""Host-timed breakdown of bench.py's e2e step at C4 (pinned H2D, GS(2), plan build,
Bi-CGSTAB, GMRES(30) x 300, x read back, plan close), each phase synchronised."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0812_2769_b200 as gsk  # noqa: E402
import workloads  # noqa: E402

s = workloads.generate(sys.argv[1] if len(sys.argv) > 1 else "C4")
pin = {k: torch.from_numpy(np.ascontiguousarray(s[k])).pin_memory() for k in ("row_ptr", "col", "val", "b")}
xo = torch.empty(s["n"], dtype=torch.float64).pin_memory()


def step(out):
    t = [time.perf_counter()]

    def mark(name):
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        out.setdefault(name, []).append(1e3 * (t[-1] - t[-2]))

    dev = {k: v.to("cuda", non_blocking=True) for k, v in pin.items()}
    mark("h2d")
    A = gsk.CSR(dev["row_ptr"], dev["col"], dev["val"])
    As, bs, _ = gsk.gs_scale(A, dev["b"], 2, inplace=True)
    mark("gs")
    P = gsk.Plan(As, fmt="sell", sell_index=os.environ.get("GSK_SELL_INDEX", "classes"))
    mark("plan")
    x1, _, r1 = P.bicgstab(bs, tol=1e-8, maxit=10000, hist=False)
    mark("bicgstab")
    x2, _, r2 = P.gmres(bs, m=30, tol=1e-8, maxit=300, hist=False)
    mark("gmres")
    xo.copy_(x1)
    xo.copy_(x2)
    mark("d2h")
    P.close()
    mark("close")
    out.setdefault("solve_ms", []).append(r1["solve_ms"] + r2["solve_ms"])


res = {}
for _ in range(int(os.environ.get("E2E_STEPS", "3"))):
    step(res)
for k, v in res.items():
    print(f"{k:10s} " + " ".join(f"{x:8.1f}" for x in v))
