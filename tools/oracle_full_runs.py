"""Run the full-size solve matrix (workloads/full_runs.py) on the ORACLE and record each
run's outcome in tests/golden/full_runs_oracle.json.

This script calls only ``oracle/`` and ``workloads/`` (no CUDA path): the stored
values are the oracle's, so tests/test_full_parity.py can compare the GPU runs with
them on the GPU box without re-running hours of host arithmetic there.  Per run:
verdict, iteration count, restarts, breakdown_at, relres / true_relres /
true_relres_w / best_relres, first crossings of 1e-6/1e-8/1e-10, sampled history
entries, and SHA-256 digests of the whole history and of x (float64 little-endian
bytes).  Resumable: runs already in the file are skipped.

    OMP_NUM_THREADS=6 python tools/oracle_full_runs.py [C1 C2 ...]
    OMP_NUM_THREADS=6 python tools/oracle_full_runs.py --paper   # -> paper_runs_oracle.json
    OMP_NUM_THREADS=4 python tools/oracle_full_runs.py --keys C4/gs2/bicgstab,C4/gs2/gmres(30)

Several processes may run at once (disjoint runs): each save re-reads the file and
merges its own record in.
"""
import hashlib
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import workloads  # noqa: E402
from workloads import full_runs  # noqa: E402

GOLDEN = {"configs": os.path.join(ROOT, "tests", "golden", "full_runs_oracle.json"),
          "paper": os.path.join(ROOT, "tests", "golden", "paper_runs_oracle.json")}


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def record(run, x, h, rep, secs):
    return {
        **{k: run[k] for k in ("key", "config", "param", "scaling", "solver", "m", "tol", "maxit", "capped",
                               "frame")},
        "status": oracle.STATUS[rep["status"]], "iterations": rep["iterations"], "restarts": rep["restarts"],
        "breakdown_at": rep["breakdown_at"], "history_len": rep["history_len"],
        "relres": rep["relres"], "true_relres": rep["true_relres"], "true_relres_w": rep["true_relres_w"],
        "best_relres": rep["best_relres"],
        "first_below": {str(t): (int(np.argmax(h < t)) if (h < t).any() else None) for t in (1e-6, 1e-8, 1e-10)},
        "hist_samples": {str(i): float(h[i]) for i in full_runs.SAMPLE_AT if i < len(h)},
        "hist_last": float(h[-1]),
        "hist_sha256": sha(h), "x_sha256": sha(x),
        "oracle_seconds": round(secs, 1), "oracle_threads": oracle.num_threads(),
    }


def save(OUT, key, rec):
    db = json.load(open(OUT)) if os.path.exists(OUT) else \
        {"_doc": __doc__.split("\n\n")[0], "host": platform.processor() or platform.machine(), "runs": {}}
    db["runs"][key] = rec
    tmp = f"{OUT}.{os.getpid()}.tmp"
    with open(tmp, "w") as f:
        json.dump(db, f, indent=1, sort_keys=True)
    os.replace(tmp, OUT)


def main(names, which="configs", keys=None):
    OUT = GOLDEN[which]
    db = {"_doc": __doc__.split("\n\n")[0], "host": platform.processor() or platform.machine(), "runs": {}}
    if os.path.exists(OUT):
        db = json.load(open(OUT))
    matrix = full_runs.runs() if which == "configs" else full_runs.paper_runs()
    todo = [r for r in matrix if (not names or r["config"] in names) and r["key"] not in db["runs"]]
    if keys:  # explicit runs, in the order given
        by_key = {r["key"]: r for r in todo}
        todo = [by_key[k] for k in keys if k in by_key]
    cache = {}
    for run in todo:
        cfg = (run["config"], run["param"])
        if cache.get("name") != cfg:
            cache = {"name": cfg, "s": workloads.generate(run["config"], param=run["param"])}
        s = cache["s"]
        if run["scaling"] not in cache:
            if run["scaling"] == "none":
                cache["none"] = (s["val"], s["b"], None)
            else:
                cache[run["scaling"]] = oracle.gs_scale(s["row_ptr"], s["val"], s["b"], run["scaling"])
        if 2 not in cache:
            cache[2] = oracle.gs_scale(s["row_ptr"], s["val"], s["b"], 2)
        val, b, dp = cache[run["scaling"]]
        w = None
        if run["frame"] == "gs2":  # GS(2)-frame stopping weights w = d2 / d_applied
            d2 = cache[2][2]
            w = d2 if dp is None else d2 / dp
        t0 = time.time()
        if run["solver"] == "bicgstab":
            x, h, rep = oracle.bicgstab(s["row_ptr"], s["col"], val, b, run["tol"], run["maxit"], weights=w)
        else:
            # frame weights only enter GMRES's reported true_relres_w (reading B2)
            x, h, rep = oracle.gmres(s["row_ptr"], s["col"], val, b, run["m"], run["tol"], run["maxit"], weights=w)
        rec = record(run, x, h, rep, time.time() - t0)
        print(json.dumps({k: rec[k] for k in ("key", "status", "iterations", "oracle_seconds")}), flush=True)
        save(OUT, run["key"], rec)


if __name__ == "__main__":
    args = sys.argv[1:]
    keys = None
    if "--keys" in args:
        i = args.index("--keys")
        keys = args[i + 1].split(",")
        del args[i:i + 2]
    main([a for a in args if a != "--paper"], "paper" if "--paper" in args else "configs", keys)
