"""Full-size run-to-verdict parity, GPU vs oracle, on the five BASELINE.json configs
(PAPER.md:299-309 for the stopping protocol).

The oracle's outcomes come from tests/golden/full_runs_oracle.json (written by
tools/oracle_full_runs.py, which calls only oracle/); this script runs the same
solves through the C-ABI on the GPU (GS on the device, SELL-C-32-256 plan, default
engine) and compares verdict, counts, residual reports and the SHA-256 of the whole
history and of x.  Writes profiles/r02_full_parity.json (argv[1] overrides) with
both sides per run and an ``equal`` flag.

    python tools/full_parity.py [out.json] [C1 C2 ...]
    python tools/full_parity.py --paper      # the paper's workloads -> r02_paper_parity.json
    python tools/full_parity.py --plain ...  # plain SELL slots instead of the row-class dictionary
"""
import hashlib
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_0812_2769_b200 as gsk  # noqa: E402
import workloads  # noqa: E402
from workloads import full_runs  # noqa: E402

GOLDEN = {"configs": os.path.join(ROOT, "tests", "golden", "full_runs_oracle.json"),
          "paper": os.path.join(ROOT, "tests", "golden", "paper_runs_oracle.json")}
FIELDS = ("status", "iterations", "restarts", "breakdown_at", "history_len", "relres", "true_relres",
          "true_relres_w", "best_relres", "hist_sha256", "x_sha256")


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def golden(which="configs"):
    return json.load(open(GOLDEN[which]))["runs"] if os.path.exists(GOLDEN[which]) else {}


def gpu_run(run, cache, sell_index="classes"):
    """One run of the matrix on the GPU; `cache` holds the config's device system.
    sell_index: the plan's encoding — "classes" (the bench default: the row-class
    dictionary where the rows repeat, C1 / C3 / C4 and the paper's problems, else the
    plain SELL slots) or "plain"."""
    cfg = (run["config"], run["param"])
    if cache.get("name") != cfg:
        cache.clear()
        s = workloads.generate(run["config"], param=run["param"])
        A0 = gsk.CSR.from_system(s)
        cache.update(name=cfg, s=s, A0=A0, b=torch.tensor(s["b"], device="cuda"))
    A0, b0 = cache["A0"], cache["b"]
    for p in (2, run["scaling"]):
        if p != "none" and p not in cache:
            cache[p] = gsk.gs_scale(A0, b0, p)
    A, b, dp = (A0, b0, None) if run["scaling"] == "none" else cache[run["scaling"]]
    w = None
    if run["frame"] == "gs2":
        d2 = cache[2][2]
        w = d2 if dp is None else d2 / dp
    P = gsk.Plan(A, fmt="sell", weights=w, sell_index=sell_index)  # GMRES: the weights only enter true_relres_w
    ncls = P.num_classes()
    t0 = time.perf_counter()
    if run["solver"] == "bicgstab":
        x, h, rep = P.bicgstab(b, tol=run["tol"], maxit=run["maxit"])
    else:
        x, h, rep = P.gmres(b, m=run["m"], tol=run["tol"], maxit=run["maxit"])
    secs = time.perf_counter() - t0
    P.close()
    out = {"status": gsk.STATUS[rep["status"]], "hist_sha256": sha(h), "x_sha256": sha(x.cpu().numpy()),
           "solve_ms": rep["solve_ms"], "wall_s": round(secs, 3), "row_classes": ncls if ncls > 0 else None,
           "first_below": {str(t): (int(np.argmax(h < t)) if (h < t).any() else None) for t in (1e-6, 1e-8, 1e-10)}}
    for k in ("iterations", "restarts", "breakdown_at", "history_len", "relres", "true_relres", "true_relres_w",
              "best_relres"):
        out[k] = rep[k]
    out["hist"] = h
    return out


def compare(ref, got):
    diff = [k for k in FIELDS if ref[k] != got[k]]
    first_diff = None
    if "hist_sha256" in diff:
        h = got["hist"]
        for i, v in sorted(((int(i), v) for i, v in ref["hist_samples"].items())):
            if i >= len(h) or h[i] != v:
                first_diff = i
                break
    return diff, first_diff


def main(out_path, names, which="configs", sell_index="classes"):
    gold = golden(which)
    cache = {}
    rows = []
    for run in (full_runs.runs() if which == "configs" else full_runs.paper_runs()):
        if names and run["config"] not in names:
            continue
        ref = gold.get(run["key"])
        if ref is None:
            continue
        got = gpu_run(run, cache, sell_index)
        diff, first_diff = compare(ref, got)
        got.pop("hist")
        rows.append({"key": run["key"], "equal": not diff, "differs_in": diff, "first_sampled_diff": first_diff,
                     "capped": run["capped"], "maxit": run["maxit"], "tol": run["tol"], "frame": run["frame"],
                     "gpu": got, "oracle": {k: ref[k] for k in FIELDS + ("first_below", "oracle_seconds")}})
        print(json.dumps({k: rows[-1][k] for k in ("key", "equal", "differs_in")} |
                         {"its": got["iterations"], "status": got["status"], "gpu_ms": round(got["solve_ms"], 1)}),
              flush=True)
    with open(out_path, "w") as f:
        json.dump({"_doc": __doc__.split("\n\n")[0], "sell_index": sell_index,
                   "all_equal": all(r["equal"] for r in rows),
                   "n_runs": len(rows), "gpu": torch.cuda.get_device_name(0), "runs": rows}, f, indent=1)
    return rows


if __name__ == "__main__":
    which = "paper" if "--paper" in sys.argv else "configs"
    sidx = "plain" if "--plain" in sys.argv else "classes"
    args = [a for a in sys.argv[1:] if a not in ("--paper", "--plain")]
    out = args[0] if args and args[0].endswith(".json") else \
        os.path.join(ROOT, "profiles", "r02_full_parity.json" if which == "configs" else "r02_paper_parity.json")
    names = [a for a in args if not a.endswith(".json")]
    rows = main(out, names, which, sidx)
    sys.exit(0 if all(r["equal"] for r in rows) else 1)
