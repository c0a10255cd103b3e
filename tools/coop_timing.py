"""Device time per Bi-CGSTAB iteration of the persistent cooperative engine (engine
"coop", csrc/coop.cu) against the graph-replayed passes (engine "graph") on mid-size
systems, and the bit-identity of the two runs (history, x, verdict).

    python tools/coop_timing.py [out.json] [--cases C2:256,C2:None,...]

GSK_COOP_G caps the cooperative grid (tuning).
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0812_2769_b200 as gsk  # noqa: E402
import workloads  # noqa: E402

CASES = [("C2", 200), ("C2", 256), ("C2", 362), ("C2", None), ("C2", 724), ("C3", 48), ("C3", 64), ("C3", 80),
         ("C5", 256), ("C5", 512), ("C5", 724)]


def parse_cases(arg):
    out = []
    for c in arg.split(","):
        name, N = c.split(":")
        out.append((name, None if N == "None" else int(N)))
    return out


def main(out, cases):
    rows = []
    for name, N in cases:
        s = workloads.generate(name, N=N)
        A0 = gsk.CSR.from_system(s)
        A, b, _ = gsk.gs_scale(A0, s["b"], 2)
        res, runs = {}, {}
        for engine in ("graph", "coop"):
            P = gsk.Plan(A, fmt="sell", engine=engine, schedule="split4")
            best = None
            for _ in range(3):  # first call: graph capture / module load
                x, h, r = P.bicgstab(b, tol=1e-12, maxit=600)
                best = r["solve_ms"] if best is None else min(best, r["solve_ms"])
            res[engine] = {"iterations": r["iterations"], "status": gsk.STATUS[r["status"]], "solve_ms": best,
                           "us_per_it": 1e3 * best / max(1, r["iterations"])}
            runs[engine] = (x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x), np.asarray(h), r)
            P.close()
        (xg, hg, rg), (xc, hc, rc) = runs["graph"], runs["coop"]
        same = bool(np.array_equal(hg, hc) and np.array_equal(xg, xc) and rg["status"] == rc["status"]
                    and rg["iterations"] == rc["iterations"] and rg["true_relres"] == rc["true_relres"])
        row = {"config": name, "N": N, "n": s["n"], "bit_identical": same,
               **{f"{k}_{e}": v for e, d in res.items() for k, v in d.items()},
               "speedup_coop": res["graph"]["solve_ms"] / res["coop"]["solve_ms"]}
        print(json.dumps(row), flush=True)
        rows.append(row)
    with open(out, "w") as f:
        json.dump(rows, f, indent=1)


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--cases")]
    cs = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--cases=")]
    main(args[0] if args else "gpurun_out/coop_timing.json", parse_cases(cs[0]) if cs else CASES)
