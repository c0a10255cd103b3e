"""Full-size runs to the verdict, GPU vs oracle (north star:
"match the oracle within the stated tolerances on all five configs").

Every solve of workloads/full_runs.py — C1..C5 at BASELINE.json's full sizes,
{unscaled, GS(1), GS(2)} x {Bi-CGSTAB, GMRES(30), the config's own GMRES(m)}, the
paper's stopping protocol (relative residual < eps, at most
10,000 iterations; GS(2)-frame weights for unscaled / GS(1) Bi-CGSTAB,
PAPER.md:305-307) — is run through the C-ABI and compared with the oracle's outcome
stored in tests/golden/full_runs_oracle.json (written by tools/oracle_full_runs.py,
which calls only oracle/).  The paper's own workloads (Table 1, tbl1a, tbl4 at 80^3,
the convection sweep; tests/golden/
paper_runs_oracle.json) are compared the same way.  Runs that end in MAXIT are capped at >= 1000 iterations
on both sides.  The comparison is bit-exact: verdict, iteration
count, breakdown_at, every reported residual and the SHA-256 of the whole history
and of x.  Where the plan's row-class dictionary applies (C1, C3, C4, Problem 4)
every run is made on both encodings.
"""
import json
import os
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

from workloads import full_runs  # noqa: E402


def _gold(name):
    path = os.path.join(ROOT, "tests", "golden", name)
    return json.load(open(path))["runs"] if os.path.exists(path) else {}


RUNS = full_runs.runs() + full_runs.paper_runs()
GOLD = {**_gold("full_runs_oracle.json"), **_gold("paper_runs_oracle.json")}

_CACHE = {}


# both plan encodings where the row-class dictionary applies (C1, C3, C4 and Problem 4:
# piecewise-constant coefficients, constant velocity); the rows of C2 (node-dependent
# velocity), C5 (random field) and Problem 1 (the conservative d(du)/dx term at 128^2:
# 16384 distinct rows) do not repeat, and "classes" falls back to the plain slots
RCD = ("C1", "C3", "C4", "P4", "P4conv")
CASES = [(r, e) for r in RUNS for e in (("classes", "plain") if r["config"] in RCD else ("classes",))]


@pytest.mark.parametrize("run,enc", CASES, ids=[f"{r['key']}-{e}" for r, e in CASES])
def test_full_size_run_to_verdict(run, enc):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    if run["key"] not in GOLD:
        pytest.skip("no oracle record for this run (tools/oracle_full_runs.py)")
    import full_parity
    ref = GOLD[run["key"]]
    got = full_parity.gpu_run(run, _CACHE, enc)
    assert (got["row_classes"] is not None) == (enc == "classes" and run["config"] in RCD)
    diff, first = full_parity.compare(ref, got)
    assert not diff, {"differs_in": diff, "first_sampled_diff": first,
                      "gpu": {k: got[k] for k in ("status", "iterations", "relres")},
                      "oracle": {k: ref[k] for k in ("status", "iterations", "relres")}}
    # north-star tolerances follow from bit-equality; state them anyway
    assert abs(got["iterations"] - ref["iterations"]) <= 2 and got["status"] == ref["status"]
