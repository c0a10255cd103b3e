"""Standalone SpMV time of a row-class plan at C4 (GS(2)); with GSK_LIB pointing at a
timing-probe build (GSK_RCD_EXP) the results are wrong and only the time is meaningful."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0812_2769_b200 as gsk  # noqa: E402
import workloads  # noqa: E402

s = workloads.generate(sys.argv[1] if len(sys.argv) > 1 else "C4")
A = gsk.CSR.from_system(s)
As, bs, _ = gsk.gs_scale(A, s["b"], 2)
P = gsk.Plan(As, fmt="sell", sell_index="classes")
x = torch.tensor(workloads.uniform(s["n"], 9, 9), device="cuda")
y = torch.empty_like(x)
for _ in range(5):
    P.spmv(x, y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(100):
    P.spmv(x, y)
e1.record()
torch.cuda.synchronize()
print(os.environ.get("GSK_LIB", "default").split("/")[-1], "classes", P.num_classes(), "slots", P.num_slots(),
      "spmv ms", round(e0.elapsed_time(e1) / 100, 4))
