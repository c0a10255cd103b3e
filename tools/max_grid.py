"""Largest grids on one B200 (SURVEY §8(f) f4's motivation: grids beyond 256³).

    python tools/max_grid.py [N ...]        (default 384 512)

C4's stencil and coefficient recipe at N³ rows (512³: 134 M rows, 939 M nonzeros,
int32 indices still suffice): GS(2) bit-exact against the oracle, the first 3
Bi-CGSTAB iterations and 2 GMRES(30) steps bit-exact against the oracle, then the
device time of 40 Bi-CGSTAB iterations and 60 GMRES(30) iterations, on the plan's row
classes (GSK_SELL_INDEX=plain: on the SELL slots).  Prints one JSON line per N.  (Test infrastructure: calls the oracle.)
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_0812_2769_b200 as gsk  # noqa: E402
import workloads  # noqa: E402


def same(g, o):
    xg, hg, rg = g
    xo, ho, ro = o
    return (np.array_equal(xg.cpu().numpy(), xo) and np.array_equal(hg, ho)
            and rg["iterations"] == ro["iterations"])


def run(N):
    t0 = time.time()
    s = workloads.generate("C4", N=N)
    n, nnz = s["n"], s["nnz"]
    tgen = time.time() - t0
    A = gsk.CSR.from_system(s)
    As, bs, _ = gsk.gs_scale(A, s["b"], 2)
    vo, bo, _ = oracle.gs_scale(s["row_ptr"], s["val"], s["b"], 2)
    gs_ok = bool(np.array_equal(As.val.cpu().numpy(), vo) and np.array_equal(bs.cpu().numpy(), bo))
    P = gsk.Plan(As, fmt="sell", sell_index=os.environ.get("GSK_SELL_INDEX", "classes"))
    ncls = P.num_classes()
    bicg_ok = same(P.bicgstab(bs, tol=1e-8, maxit=3), oracle.bicgstab(s["row_ptr"], s["col"], vo, bo, 1e-8, 3))
    gm_ok = same(P.gmres(bs, m=30, tol=1e-8, maxit=2), oracle.gmres(s["row_ptr"], s["col"], vo, bo, 30, 1e-8, 2))
    del A, s, vo
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = {"N": N, "n": n, "nnz": nnz, "gen_s": round(tgen, 1), "row_classes": ncls if ncls > 0 else None,
           "gs_bitexact": gs_ok,
           "bicgstab_3its_bitexact": bool(bicg_ok), "gmres_2steps_bitexact": bool(gm_ok)}
    for name, call, its in (("bicgstab", lambda: P.bicgstab(bs, tol=1e-30, maxit=40), 40),
                            ("gmres30", lambda: P.gmres(bs, m=30, tol=1e-30, maxit=60), 60)):
        call()
        e0.record()
        _, _, rep = call()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        out[name + "_its_per_s"] = round(rep["iterations"] / (ms / 1e3), 1)
    # bytes: Bi-CGSTAB split schedule 2 B_A + 19 vectors per iteration
    BA = 2 * n if ncls > 0 else 12 * nnz + 4 * (n + 1)  # row classes: class ids instead of slot data
    out["bicgstab_gbps_19vec"] = round(out["bicgstab_its_per_s"] * (2 * BA + 19 * 8 * n) / 1e9, 1)
    free, total = torch.cuda.mem_get_info()
    out["gpu_mem_used_gb"] = round((total - free) / 2**30, 1)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    for N in [int(a) for a in sys.argv[1:]] or [384, 512]:
        run(N)
