"""GS(2) on the C4 system, three calls (ncu target for gs_kernel):
ncu --set full -k regex:gs_kernel --launch-skip 2 -c 1 python tools/prof_gs.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0812_2769_b200 as gsk  # noqa: E402
import workloads  # noqa: E402

s = workloads.generate(sys.argv[1] if len(sys.argv) > 1 else "C4")
A = gsk.CSR.from_system(s)
b = torch.tensor(s["b"], device="cuda")
out = (torch.empty_like(A.val), torch.empty_like(b), torch.empty_like(b))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for p in (2, 2, 2, 1):
    e0.record()
    gsk.gs_scale(A, b, p, out=out)
    e1.record()
    torch.cuda.synchronize()
    print("GS(%d) %.3f ms" % (p, e0.elapsed_time(e1)))
for _ in range(3):
    e0.record()
    gsk.gs_scale_sym(A, b, 2)
    e1.record()
    torch.cuda.synchronize()
    print("two-sided GS(2) %.3f ms" % e0.elapsed_time(e1))
