"""The full-size run matrix: which solves are
run to their verdict on BOTH sides — the oracle (tools/oracle_full_runs.py, CPU) and
the CUDA path (tests/test_full_parity.py, tools/full_parity.py) — on the five
BASELINE.json configs at full size.

Pure recipe data (no arithmetic of the method): config, scaling, solver, restart,
tolerance, iteration cap and stopping frame.

* Stopping follows the paper's protocol: relative residual < eps,
  at most 10,000 iterations (C1: 2000, BASELINE.json), eps = the config's tightest
  tolerance (iterates do not depend on eps, reading B11).
* Unscaled and GS(1) Bi-CGSTAB runs stop in the GS(2) frame:
  weights w = d2 / d_applied.  GMRES runs stop on their least-squares estimate in
  the solved frame (reading B2) and report the GS(2)-frame true residual.
* Runs that end in MAXIT at 10,000 iterations are capped (``cap``) at >= 1000
  iterations on both sides, as SURVEY §8(d.5) allows: the oracle at full length
  would take hours on the host (a non-converging GMRES(30) at C4 moves ~100 TB).
  Both sides then run to the same cap and must agree bit for bit, verdict included.
"""
from __future__ import annotations

# (config, scaling, solver, m, cap or None)
_MATRIX = [
    # C1: 32^2, GS(2) vs unscaled, Bi-CGSTAB + GMRES(20) (+ GMRES(30), reading B14)
    ("C1", "none", "bicgstab", None, None), ("C1", "none", "gmres", 20, None), ("C1", "none", "gmres", 30, None),
    ("C1", 2, "bicgstab", None, None), ("C1", 2, "gmres", 20, None), ("C1", 2, "gmres", 30, None),
    # C2: 512^2, GS(1) and GS(2) (+ unscaled), Bi-CGSTAB + GMRES(30), tol 1e-10
    ("C2", 2, "bicgstab", None, None), ("C2", 1, "bicgstab", None, None), ("C2", "none", "bicgstab", None, None),
    ("C2", 2, "gmres", 30, None), ("C2", 1, "gmres", 30, None), ("C2", "none", "gmres", 30, None),
    # C3: 128^3, GS(2) (+ unscaled)
    ("C3", 2, "bicgstab", None, None), ("C3", 2, "gmres", 30, None),
    ("C3", "none", "bicgstab", None, 2000), ("C3", "none", "gmres", 30, 2000),
    # C5: 2048^2 permuted, {none, GS(1), GS(2)} x {Bi-CGSTAB, GMRES(50), GMRES(30)}; all MAXIT
    ("C5", 2, "bicgstab", None, 2000), ("C5", 1, "bicgstab", None, 2000), ("C5", "none", "bicgstab", None, 2000),
    ("C5", 2, "gmres", 50, 1000), ("C5", 1, "gmres", 50, 1000), ("C5", "none", "gmres", 50, 1000),
    ("C5", 2, "gmres", 30, 1000),
    # C4: 256^3, the headline config: GS(2) runs to the verdict; unscaled capped
    ("C4", 2, "bicgstab", None, None), ("C4", "none", "bicgstab", None, 1000),
    ("C4", "none", "gmres", 30, 1000), ("C4", 2, "gmres", 30, None),
]


# The paper's own workloads: Table 1 / tbl1a (Problem 1, 128^2,
# PAPER.md:375-384, 422-429), tbl4 (Problem 4, 80^3, D = 1e4 / 1e6)
# and the convection sweep "limit" (Problem 4, 40^3).  Every run
# goes to 1e-10 (the paper's tightest goal).  Unscaled Bi-CGSTAB
# stops in the GS(2) frame; GMRES(10) stops on its least-squares
# estimate in the solved frame and REPORTS the GS(2)-frame true residual
# (true_relres_w; frame weights do not change a GMRES run, reading B2).
# (workload, param, scaling, solver, m, maxit)
_PAPER = [(w, None, sc, sv, m, 10000) for w in ("P1", "P1cont") for sc in ("none", 2)
          for sv, m in (("bicgstab", None), ("gmres", 10))] + \
         [("P4", D, sc, sv, m, 2000) for D in (1e4, 1e6) for sc in ("none", 2)
          for sv, m in (("bicgstab", None), ("gmres", 10))] + \
         [("P4conv", cv, sc, "bicgstab", None, 10000) for cv in (100.0, 200.0, 500.0, 1000.0) for sc in ("none", 2)]


def key(r: dict) -> str:
    s = "gs%s" % r["scaling"] if r["scaling"] != "none" else "none"
    w = r["config"] + (f"[{r['param']:g}]" if r.get("param") is not None else "")
    return f"{w}/{s}/{r['solver']}" + (f"({r['m']})" if r["m"] else "")


def runs() -> list[dict]:
    from . import CONFIGS
    out = []
    for cfg, scaling, solver, m, cap in _MATRIX:
        c = CONFIGS[cfg]
        out.append({"config": cfg, "param": None, "scaling": scaling, "solver": solver, "m": m,
                    "tol": min(c.tols or (c.tol,)), "maxit": min(c.maxit, cap or c.maxit),
                    "capped": cap is not None,
                    "frame": "gs2" if (solver == "bicgstab" and scaling != 2) else "solved"})
    for r in out:
        r["key"] = key(r)
    return out


def paper_runs() -> list[dict]:
    out = []
    for wl, param, scaling, solver, m, maxit in _PAPER:
        r = {"config": wl, "param": param, "scaling": scaling, "solver": solver, "m": m, "tol": 1e-10,
             "maxit": maxit, "capped": False, "frame": "gs2" if scaling != 2 else "solved",
             "report_frame": "gs2" if scaling != 2 else "solved"}
        r["key"] = key(r)
        out.append(r)
    return out


# history entries recorded in the golden file (besides the SHA-256 of the whole history)
SAMPLE_AT = (1, 2, 5, 10, 20, 50, 100, 200, 500, 1000, 1500, 2000, 3000, 5000, 7500, 10000)
