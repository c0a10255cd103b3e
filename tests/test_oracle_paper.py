"""Oracle pinned to the paper's printed tables (tests/golden/paper_tables.json).

The paper ran AZTEC (CGS2 GMRES, Pentium IV); our oracle follows DESIGN.md's
readings (MGS, face-midpoint k, h^2 scaling, GS(2)-frame stopping B2).  Bands:
GMRES is insensitive to rounding, so its counts must land within
2% of the paper; Bi-CGSTAB's residual history is chaotic on these systems, so its
counts get a 10% band (SURVEY §4.2 reproduced every one within 10% with textbook
numpy solvers); verdicts ("no conv.", "---", stagnation level) must match.

One entry keeps 20%: tbl1a unscaled Bi-CGSTAB at 1e-7 (paper 224, oracle 190).  That
history falls in a staircase — 2.8e-7 at iteration 188, 5.8e-8 at 190, back up to
2.5e-7 at 215, 1.8e-8 at 218 — so which step first crosses 1e-7 depends on the
rounding of the whole run: changing only the dot-product summation order moves such
counts by tens of iterations.  `test_tbl1a_staircase` pins that
explanation.
"""
import json
import os

import numpy as np
import pytest

import oracle
import workloads

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_tables.json")))
TOLS = GOLD["tolerances"]["eps"]


def first_crossings(h):
    return [int(np.argmax(h < t)) if (h < t).any() else None for t in TOLS]


def scaled(name, N=None, param=None):
    s = workloads.generate(name, N=N, param=param)
    vo, bo, d = oracle.gs_scale(s["row_ptr"], s["val"], s["b"], 2)
    return s, vo, bo, d


def check(ours, paper, band):
    bands = band if isinstance(band, (list, tuple)) else [band] * len(paper)
    for o, p, bd in zip(ours, paper, bands):
        if p is None:
            assert o is None, (ours, paper)
        else:
            assert o is not None and abs(o - p) <= bd * p, (ours, paper)


def test_tbl1_problem1_bicgstab():
    """Table 1: Bi-CGSTAB fails unscaled; GS(2) converges 91/299/361.
    Stopping is always measured on the GS(2)-scaled system."""
    s, vo, bo, d = scaled("P1")
    _, h, rep = oracle.bicgstab(s["row_ptr"], s["col"], s["val"], s["b"], 1e-10, 10000, weights=d)
    assert first_crossings(h) == [None, None, None] and rep["status"] != 0
    _, h, rep = oracle.bicgstab(s["row_ptr"], s["col"], vo, bo, 1e-10, 10000)
    check(first_crossings(h), GOLD["tbl1"]["bicgstab_gs2"], 0.10)


@pytest.mark.slow
@pytest.mark.parametrize("orth", ["mgs", "cgs2"])
def test_tbl1_problem1_gmres(orth):
    """Table 1: GMRES(10) stalls near 3.8e-2 unscaled; with GS(2)
    it reaches 1e-4 at 265 and stalls at 1.1e-5 — with MGS and with the paper's own
    double classical Gram-Schmidt."""
    s, vo, bo, d = scaled("P1")
    _, h, rep = oracle.gmres(s["row_ptr"], s["col"], vo, bo, 10, 1e-10, 10000, orth=orth)
    assert first_crossings(h)[0] == GOLD["tbl1"]["gmres10_gs2"][0]
    stall = rep["best_relres"]
    assert first_crossings(h)[1] is None
    assert 0.5 * GOLD["tbl1"]["gmres10_gs2_stall"] < stall < 2 * GOLD["tbl1"]["gmres10_gs2_stall"]
    _, h, rep = oracle.gmres(s["row_ptr"], s["col"], s["val"], s["b"], 10, 1e-10, 3000, weights=d)
    assert first_crossings(h)[0] is None
    assert 1e-2 < rep["true_relres_w"] < 1e-1  # paper 3.8e-2 in the GS(2) frame


@pytest.mark.slow
def test_tbl1a_continuous_problem1():
    """Table tbl1a, a = b = 1000 everywhere."""
    s, vo, bo, d = scaled("P1cont")
    g = GOLD["tbl1a"]
    for orth in ("mgs", "cgs2"):
        _, h, _ = oracle.gmres(s["row_ptr"], s["col"], vo, bo, 10, 1e-10, 7000, orth=orth)
        check(first_crossings(h), g["gmres10_gs2"], 0.02)
    _, h, _ = oracle.gmres(s["row_ptr"], s["col"], s["val"], s["b"], 10, 1e-10, 7000)
    check(first_crossings(h), g["gmres10_unscaled"], 0.02)
    _, h, _ = oracle.bicgstab(s["row_ptr"], s["col"], vo, bo, 1e-10, 10000)
    check(first_crossings(h), g["bicgstab_gs2"], 0.10)
    _, h, _ = oracle.bicgstab(s["row_ptr"], s["col"], s["val"], s["b"], 1e-10, 10000, weights=d)
    check(first_crossings(h), g["bicgstab_unscaled"], [0.10, 0.20, 0.10])


def test_tbl1a_staircase():
    """The one 20% band above: the unscaled continuous-Problem-1 Bi-CGSTAB history
    (GS(2) frame) crosses 1e-7 in jumps, with a relapse above 1e-7 between the
    oracle's crossing (190) and the paper's (224), so a rounding-level change of the
    run moves the first crossing by a whole step of the staircase."""
    s, vo, bo, d = scaled("P1cont")
    _, h, _ = oracle.bicgstab(s["row_ptr"], s["col"], s["val"], s["b"], 1e-10, 10000, weights=d)
    k = first_crossings(h)[1]
    assert h[k - 2] > 2.5e-7 and h[k] < 6e-8        # 4x down across 1e-7 in two steps
    assert (h[k:224] > 1e-7).any()                  # a relapse above 1e-7 before 224
    assert h[224] < 1e-7


@pytest.mark.slow
@pytest.mark.parametrize("D", [1e4, 1e6])
def test_tbl4_problem4(D):
    """Table tbl4, 80^3: Bi-CGSTAB '---' unscaled, GS(2)
    112/262/406 (D=1e4) and 111/160/374 (D=1e6); GS(2)+GMRES(10) 208 / 207, 286."""
    s, vo, bo, d = scaled("P4", param=D)
    g = GOLD["tbl4"]
    key = "D1e4" if D == 1e4 else "D1e6"
    _, h, rep = oracle.bicgstab(s["row_ptr"], s["col"], s["val"], s["b"], 1e-10, 1000, weights=d)
    assert first_crossings(h) == [None, None, None]
    _, h, rep = oracle.bicgstab(s["row_ptr"], s["col"], vo, bo, 1e-10, 1000)
    check(first_crossings(h), g["bicgstab_gs2_" + key], 0.10)
    _, h, rep = oracle.gmres(s["row_ptr"], s["col"], vo, bo, 10, 1e-10, 400)
    check(first_crossings(h), g["gmres10_gs2_" + key], 0.02)
