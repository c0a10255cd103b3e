"""Run every BASELINE.json config on the GPU: {none, GS(1), GS(2), two-sided D^1/2 A D^1/2
with p = 2} x {Bi-CGSTAB, GMRES(m)}.

For each run: iterations to each tolerance (first crossing of the history), verdict,
best relative residual, device time of the solve and time to the tightest tolerance
reached, with and without GS (the north star's "time-to-1e-8 with/without GS").
Unscaled and GS(1) Bi-CGSTAB runs stop in the GS(2) frame as the paper does
(PAPER.md:305-307); GMRES runs stop in the solved frame and report the GS(2)-frame
true residual.  Writes JSON and a markdown table (argv[1] prefix).

    python tools/run_configs.py profiles/r01_configs [C1 C2 ...]
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0812_2769_b200 as gsk  # noqa: E402
import workloads  # noqa: E402


# plan encoding: the row-class dictionary where the rows repeat (the bench default), else
# (and with GSK_SELL_INDEX=plain) the plain SELL slots
SELL_INDEX = os.environ.get("GSK_SELL_INDEX", "classes")


def first(h, tol):
    idx = np.flatnonzero(h < tol)
    return int(idx[0]) if idx.size else None


def run(name, maxit_gmres=None):
    c = workloads.CONFIGS[name]
    s = workloads.generate(name)
    fmt = "sell"  # SELL-C-32-256 on every config (faster than CSR everywhere)
    A0 = gsk.CSR.from_system(s)
    _, _, d2 = gsk.gs_scale(A0, s["b"], 2)
    gsk.gs_scale(A0, s["b"], 1)  # warm-up: module load / allocator pools out of the timings
    rows = []
    tols = c.tols or (c.tol,)
    for scaling in ("none", 1, 2, "sym2"):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        A = gsk.CSR.from_system(s)
        b = torch.tensor(s["b"], device="cuda")
        w = d2
        gs_ms = 0.0
        if scaling == "sym2":  # PAPER.md:245-251; GS(2) frame: D r = D^1/2 r_sym -> w = s
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            A, b, sv = gsk.gs_scale_sym(A, b, 2)
            e1.record()
            torch.cuda.synchronize()
            gs_ms = e0.elapsed_time(e1)
            w = sv
        elif scaling != "none":
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            A, b, dp = gsk.gs_scale(A, b, scaling, inplace=True)
            e1.record()
            torch.cuda.synchronize()
            gs_ms = e0.elapsed_time(e1)
            w = None if scaling == 2 else d2 / dp
        for solver, m in (("bicgstab", None), ("gmres", 30), ("gmres", c.m)):
            if solver == "gmres" and m == 30 and c.m == 30 and any(r["solver"] == "gmres(30)" and
                                                                   r["scaling"] == str(scaling) for r in rows):
                continue
            P = gsk.Plan(A, fmt="sell", weights=w if solver == "bicgstab" else None, sell_index=SELL_INDEX)
            ncls = P.num_classes()
            maxit = c.maxit if solver == "bicgstab" else (maxit_gmres or c.maxit)
            if solver == "bicgstab":
                x, h, rep = P.bicgstab(b, tol=min(tols), maxit=maxit)
            else:
                x, h, rep = P.gmres(b, m=m, tol=min(tols), maxit=maxit)
            tr2 = None
            if solver == "gmres" and scaling != 2:
                # report the GS(2)-frame true residual
                Pw = gsk.Plan(A, fmt="sell")
                r0 = Pw.residual_norm(b, torch.zeros_like(b), w)
                tr2 = Pw.residual_norm(b, x, w) / r0
            its = {str(t): first(h, t) for t in tols}
            ms = rep["solve_ms"]
            n, nnz = s["n"], s["nnz"]
            ba = 2 * n if ncls > 0 else 12 * nnz + 4 * (n + 1)  # class ids instead of slot data
            # algorithmic bytes per iteration: Bi-CGSTAB split schedule 2 B_A + 19 vectors;
            # MGS GMRES(m) averaged over a cycle: step j moves B_A + (4j + 3) vectors (S_j, h_1j, j-1 M, L),
            # the restart (X, R) B_A + (m + 5) vectors per m steps
            bpi = (2 * ba + 19 * 8 * n) if solver == "bicgstab" else \
                (ba * (1 + 1 / m) + (2 * (m + 1) + 3 + (m + 5) / m) * 8 * n)
            its_done = max(rep["iterations"], 1)
            rows.append({
                "config": name, "scaling": str(scaling), "solver": f"{solver}" + (f"({m})" if m else ""),
                "row_classes": ncls if ncls > 0 else None,
                "status": gsk.STATUS[rep["status"]], "iterations": rep["iterations"], "its_to_tol": its,
                "best_relres": rep["best_relres"], "true_relres": rep["true_relres"],
                "true_relres_gs2_frame": tr2 if tr2 is not None else rep["true_relres_w"],
                "solve_ms": ms, "gs_ms": gs_ms,
                "ms_per_iter": ms / max(rep["iterations"], 1),
                "gbps_model": bpi * its_done / (ms / 1e3) / 1e9 if ms else None,
                "time_to_tightest_ms": (gs_ms + ms) if rep["status"] == 0 else None,
            })
            print(json.dumps(rows[-1]), flush=True)
            P.close()
    return rows


def markdown(rows):
    out = ["| config | scaling | solver | classes | verdict | its to tol | best rel-res | solve ms | ms/it | GB/s (model) | GS ms |",
           "|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        its = ", ".join(f"{k}: {v if v is not None else '—'}" for k, v in r["its_to_tol"].items())
        out.append(f"| {r['config']} | {r['scaling']} | {r['solver']} | {r.get('row_classes') or '—'} | "
                   f"{r['status']} ({r['iterations']}) | {its} | "
                   f"{r['best_relres']:.2e} | {r['solve_ms']:.1f} | {r['ms_per_iter']:.3f} | {r['gbps_model']:.0f} | "
                   f"{r['gs_ms']:.2f} |")
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    prefix = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/configs"
    names = sys.argv[2:] or ["C1", "C2", "C3", "C4", "C5"]
    allrows = []
    for nm in names:
        allrows += run(nm)
    with open(prefix + ".json", "w") as f:
        json.dump(allrows, f, indent=1)
    with open(prefix + ".md", "w") as f:
        f.write(markdown(allrows))
    print(markdown(allrows))
