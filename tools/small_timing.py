"""Device time per iteration of the on-chip single-CTA solvers (engine "small") vs the
graph-replayed passes (engine "graph") on small systems (C1 and small C2/C3/C5 grids).

    python tools/small_timing.py [out.json]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0812_2769_b200 as gsk  # noqa: E402
import workloads  # noqa: E402

CASES = [("C1", None, 20), ("C2", 40, 30), ("C2", 64, 30), ("C3", 16, 30), ("C5", 64, 50), ("C5", 96, 30),
         ("P1", None, 10), ("C3", 24, 30), ("C3", 32, 30), ("C2", 200, 30), ("P4conv", None, 10)]


def main(out):
    rows = []
    for name, N, m in CASES:
        s = workloads.generate(name, N=N)
        A0 = gsk.CSR.from_system(s)
        A, b, _ = gsk.gs_scale(A0, s["b"], 2)
        for solver in ("bicgstab", "gmres"):
            res = {}
            for engine in ("small", "cluster", "graph"):
                if engine == "small" and s["n"] > 4096:
                    continue
                P = gsk.Plan(A, engine=engine)
                best = None
                for _ in range(3):  # first call: graph capture / module load
                    if solver == "bicgstab":
                        x, h, r = P.bicgstab(b, tol=1e-8, maxit=2000)
                    else:
                        x, h, r = P.gmres(b, m=m, tol=1e-8, maxit=2000)
                    best = r["solve_ms"] if best is None else min(best, r["solve_ms"])
                res[engine] = {"iterations": r["iterations"], "status": gsk.STATUS[r["status"]], "solve_ms": best,
                               "us_per_it": 1e3 * best / max(1, r["iterations"])}
                P.close()
            row = {"config": name, "N": N, "n": s["n"], "solver": solver + (f"({m})" if solver == "gmres" else ""),
                   **{f"{k}_{e}": v for e, d in res.items() for k, v in d.items()},
                   "speedup_cluster": res["graph"]["solve_ms"] / res["cluster"]["solve_ms"]}
            print(json.dumps(row), flush=True)
            rows.append(row)
    with open(out, "w") as f:
        json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/small_timing.json")
