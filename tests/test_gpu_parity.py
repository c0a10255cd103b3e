"""GPU <-> oracle parity through the C-ABI (north-star contract).

Under the arithmetic contract the CUDA path and the oracle are bit-identical, so
every comparison is exact (==): integer work, GS values, SpMV, histories, x,
iteration counts and verdicts.  `tolerance_report` additionally evaluates the
north-star tolerances (GS <= 2 ulp, per-iteration relres <= 1e-9 relative over the
first 50 iterations, iterations +-2, x <= 1e-7 relative) so that a contract slip
is distinguishable from a tolerance failure.
"""
import json
import os

import numpy as np
import pytest

import oracle
import workloads

pytestmark = pytest.mark.gpu

gsk = pytest.importorskip("paper_0812_2769_b200")
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # collected on CPU boxes but never run there
    pytest.skip("needs a CUDA device", allow_module_level=True)


def ulps(a, b):
    a = np.ascontiguousarray(a, np.float64).view(np.int64)
    b = np.ascontiguousarray(b, np.float64).view(np.int64)
    return int(np.abs(a - b).max()) if a.size else 0


def cpu(t):
    return t.detach().cpu().numpy() if hasattr(t, "detach") else np.asarray(t)


def tolerance_report(h_gpu, h_orc, x_gpu, x_orc, it_gpu, it_orc):
    k = min(len(h_gpu), len(h_orc), 51)
    rel = np.abs(h_gpu[:k] - h_orc[:k]) / np.maximum(np.abs(h_orc[:k]), 1e-300)
    assert rel.max() <= 1e-9
    assert abs(it_gpu - it_orc) <= 2
    xs = np.linalg.norm(x_orc)
    assert np.linalg.norm(x_gpu - x_orc) <= 1e-7 * (xs if xs > 0 else 1.0)


def same(a, b):
    """== with NaN equal to NaN (a DIVERGED run's values; NaN payloads differ between
    x86 and the GPU, so bit patterns are not compared)."""
    return a == b or (a != a and b != b)


def assert_same_solve(g, o):
    xg, hg, rg = g
    xo, ho, ro = o
    xg = cpu(xg)
    for k in ("status", "iterations", "history_len", "breakdown_at", "restarts"):
        assert rg[k] == ro[k], (k, rg, ro)
    assert np.array_equal(hg, ho, equal_nan=True), np.flatnonzero(hg != ho)[:5]
    assert np.array_equal(xg, xo, equal_nan=True)
    for k in ("relres", "best_relres", "true_relres", "true_relres_w"):
        assert same(rg[k], ro[k]), (k, rg[k], ro[k])
    if ro["status"] != 3:
        tolerance_report(hg, ho, xg, xo, rg["iterations"], ro["iterations"])


CASES = [("C1", None), ("C2", 100), ("C2", 128), ("C3", 20), ("C4", 24), ("C5", 96), ("P1", 64)]


# ---------------------------------------------------------------- GS(p)
@pytest.mark.parametrize("p", [1, 2])
def test_gs_zero_rows_outputs(p):
    """Zero rows (PAPER.md:207-208 assumes none; reading G5): GSK_E_ZERO_ROW names the
    smallest one, and the GPU's outputs are fixed as gsk.h states — d_i = 0, the row's
    values and b_i stay zero, every other row is scaled exactly as the oracle scales it
    (GS is row-local: the oracle is run with the zero rows given a placeholder value)."""
    s = workloads.generate("C1")
    rp, val, b = s["row_ptr"], s["val"].copy(), s["b"].copy()
    zero = [700, 3, 517]
    for r in zero:
        val[rp[r]:rp[r + 1]] = 0.0
    A = gsk.CSR(rp, s["col"], val)
    vout = torch.full((val.size,), 7.0, dtype=torch.float64, device="cuda")
    bout = torch.full((s["n"],), 7.0, dtype=torch.float64, device="cuda")
    dout = torch.full((s["n"],), 7.0, dtype=torch.float64, device="cuda")
    with pytest.raises(gsk.GskError) as e:
        gsk.gs_scale(A, b, p, out=(vout, bout, dout))
    assert e.value.code == -2 and e.value.bad_row == 3  # GSK_E_ZERO_ROW
    ph = val.copy()
    for r in zero:
        ph[rp[r]:rp[r + 1]] = 1.0
    vo, bo, do = oracle.gs_scale(rp, ph, b, p)
    vg, bg, dg = cpu(vout), cpu(bout), cpu(dout)
    zmask = np.zeros(s["n"], bool)
    zmask[zero] = True
    emask = np.repeat(zmask, np.diff(rp))
    assert np.array_equal(vg[~emask], vo[~emask]) and np.array_equal(bg[~zmask], bo[~zmask])
    assert np.array_equal(dg[~zmask], do[~zmask])
    assert np.all(vg[emask] == 0.0) and np.all(bg[zmask] == 0.0) and np.all(dg[zmask] == 0.0)


@pytest.mark.parametrize("name,N", CASES + [("C4", None), ("C5", None)])
@pytest.mark.parametrize("p", [1, 2, 3])
def test_gs_scale_parity(name, N, p):
    s = workloads.generate(name, N=N)
    A = gsk.CSR.from_system(s)
    As, bs, d = gsk.gs_scale(A, s["b"], p)
    vo, bo, do = oracle.gs_scale(s["row_ptr"], s["val"], s["b"], p)
    if p in (1, 2):  # AC-4: bit-exact
        assert np.array_equal(cpu(As.val), vo)
        assert np.array_equal(cpu(bs), bo)
        assert np.array_equal(cpu(d), do)
    else:  # pow() is libm-dependent: north-star 2 ulp on the norm, a few on the products
        assert ulps(1.0 / cpu(d), 1.0 / do) <= 2
        assert ulps(cpu(As.val), vo) <= 4
    # in place gives the same bits
    A2 = gsk.CSR.from_system(s)
    b2 = torch.tensor(s["b"], device="cuda")
    gsk.gs_scale(A2, b2, p, inplace=True)
    assert np.array_equal(cpu(A2.val), cpu(As.val)) and np.array_equal(cpu(b2), cpu(bs))


def test_gs_errors():
    s = workloads.generate("C2", N=40)
    val = s["val"].copy()
    for r in (700, 33, 1599):
        val[s["row_ptr"][r]:s["row_ptr"][r + 1]] = 0.0
    A = gsk.CSR(s["row_ptr"], s["col"], val)
    with pytest.raises(gsk.GskError) as ei:
        gsk.gs_scale(A, s["b"], 2)
    assert ei.value.code == -2 and ei.value.bad_row == 33
    with pytest.raises(gsk.GskError) as ei:
        gsk.gs_scale(gsk.CSR.from_system(s), s["b"], 0)
    assert ei.value.code == -1


# ---------------------------------------------------------------- SpMV, dot, SELL
@pytest.mark.parametrize("name,N", CASES + [("C4", None), ("C5", None)])
@pytest.mark.parametrize("fmt", ["csr", "sell"])
def test_spmv_parity(name, N, fmt):
    s = workloads.generate(name, N=N)
    A = gsk.CSR.from_system(s)
    P = gsk.Plan(A, fmt=fmt)
    x = workloads.uniform(s["n"], 77, 3)
    y = cpu(P.spmv(x))
    assert np.array_equal(y, oracle.spmv(s["row_ptr"], s["col"], s["val"], x))
    if fmt == "csr":
        assert np.array_equal(cpu(gsk.spmv(A, x)), y)


def test_spmv_long_rows_fallback():
    # rows longer than the shared-memory stage (2048 entries per 256 rows) take the
    # direct path; results must not change
    rng = np.random.default_rng(8)
    n = 700
    lens = rng.integers(0, 40, n)
    lens[:256] = 30
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    col = np.concatenate([np.sort(rng.choice(n, l, replace=False)) for l in lens]).astype(np.int32)
    val = rng.standard_normal(rp[-1])
    x = rng.standard_normal(n)
    for fmt in ("csr", "sell"):
        y = cpu(gsk.Plan(gsk.CSR(rp, col, val), fmt=fmt).spmv(x))
        assert np.array_equal(y, oracle.spmv(rp, col, val, x))


@pytest.mark.parametrize("name,N", [("C1", None), ("C2", 100), ("C3", 20), ("C4", None), ("C5", 300)])
def test_sell_layout_parity(name, N):
    s = workloads.generate(name, N=N)
    P = gsk.Plan(gsk.CSR.from_system(s), fmt="sell")
    g = P.sell_arrays()
    o = oracle.sell_build(s["row_ptr"], s["col"], s["val"], 32, 256)
    for k in ("chunk_ptr", "chunk_len", "scol", "sval", "roff"):
        assert np.array_equal(g[k], o[k]), k


@pytest.mark.parametrize("name,N", [("C1", None), ("C2", 100), ("C3", 20), ("C4", None), ("C5", 64)])
def test_sell_dict_parity(name, N):
    """Column-index dictionary built on the device == the oracle's encoding (integer
    bit-exact); C5's permuted system keeps plain int32 columns on both sides."""
    s = workloads.generate(name, N=N)
    P = gsk.Plan(gsk.CSR.from_system(s), fmt="sell", sell_index="dict")
    g = P.sell_dict()
    o = oracle.sell_dict(s["n"], oracle.sell_build(s["row_ptr"], s["col"], s["val"], 32, 256))
    if o is None:
        assert g is None
        return
    for k in ("dict_ptr", "dict", "sidx"):
        assert np.array_equal(g[k], o[k]), k
    # plain-index plan gives the same SpMV bits
    x = workloads.uniform(s["n"], 5, 5)
    Pp = gsk.Plan(gsk.CSR.from_system(s), fmt="sell")
    assert Pp.sell_dict() is None
    assert np.array_equal(cpu(P.spmv(x)), cpu(Pp.spmv(x)))
    vo, bo, _ = oracle.gs_scale(s["row_ptr"], s["val"], s["b"], 2)
    Pd = gsk.Plan(gsk.CSR(s["row_ptr"], s["col"], vo), fmt="sell", sell_index="dict")
    assert_same_solve(Pd.bicgstab(bo, tol=1e-8, maxit=200), oracle.bicgstab(s["row_ptr"], s["col"], vo, bo, 1e-8, 200))
    assert_same_solve(Pd.gmres(bo, m=20, tol=1e-8, maxit=60), oracle.gmres(s["row_ptr"], s["col"], vo, bo, 20, 1e-8, 60))


@pytest.mark.parametrize("n", [1, 3, 255, 256, 257, 4097, 65536, 65537, 1000003, 3000001])
def test_dot_parity(n):
    a = workloads.uniform(n, 5, 11) * np.exp(workloads.uniform(n, 6, 11, -20, 20))
    b = workloads.uniform(n, 7, 11)
    assert gsk.dot(a, b) == oracle.dot(a, b)


# ---------------------------------------------------------------- solvers
def system(name, N, scaling):
    s = workloads.generate(name, N=N)
    if scaling == "none":
        return s, s["val"], s["b"], None
    vo, bo, d = oracle.gs_scale(s["row_ptr"], s["val"], s["b"], scaling)
    return s, vo, bo, d


@pytest.mark.parametrize("name,N", CASES)
@pytest.mark.parametrize("scaling", ["none", 1, 2])
@pytest.mark.parametrize("fmt", ["csr", "sell"])
@pytest.mark.parametrize("schedule", ["fused", "split", "split4"])
def test_bicgstab_parity(name, N, scaling, fmt, schedule):
    s, val, b, _ = system(name, N, scaling)
    maxit = 600
    P = gsk.Plan(gsk.CSR(s["row_ptr"], s["col"], val), fmt=fmt, schedule=schedule, engine="graph")
    g = P.bicgstab(b, tol=1e-8, maxit=maxit)
    o = oracle.bicgstab(s["row_ptr"], s["col"], val, b, 1e-8, maxit)
    assert_same_solve(g, o)


def test_bicgstab_frame_weights():
    """Stopping in the GS(2) frame for an unscaled / GS(1) solve."""
    s = workloads.generate("P1", N=64)
    _, _, d2 = oracle.gs_scale(s["row_ptr"], s["val"], s["b"], 2)
    for p, schedule in (("none", "fused"), ("none", "split"), (1, "fused"), (1, "split")):
        if p == "none":
            val, b, w = s["val"], s["b"], d2
        else:
            val, b, d1 = oracle.gs_scale(s["row_ptr"], s["val"], s["b"], 1)
            w = d2 / d1
        P = gsk.Plan(gsk.CSR(s["row_ptr"], s["col"], val), weights=w, schedule=schedule, engine="graph")
        g = P.bicgstab(b, tol=1e-10, maxit=3000)
        o = oracle.bicgstab(s["row_ptr"], s["col"], val, b, 1e-10, 3000, weights=w)
        assert_same_solve(g, o)


@pytest.mark.parametrize("name,N", CASES)
@pytest.mark.parametrize("scaling", ["none", 2])
@pytest.mark.parametrize("m", [1, 20, 30, 50])
@pytest.mark.parametrize("orth", ["mgs", "cgs2"])
def test_gmres_parity(name, N, scaling, m, orth):
    s, val, b, _ = system(name, N, scaling)
    maxit = 400
    fmt = "sell" if name == "C4" else "csr"
    P = gsk.Plan(gsk.CSR(s["row_ptr"], s["col"], val), fmt=fmt, orth=orth, engine="graph")
    g = P.gmres(b, m=m, tol=1e-8, maxit=maxit)
    o = oracle.gmres(s["row_ptr"], s["col"], val, b, m, 1e-8, maxit, orth=orth)
    assert_same_solve(g, o)


def test_gmres_cgs2_paper_problem1():
    """GS(2) + GMRES(10) with the paper's own orthogonalisation on
    Problem 1 128x128: bit-exact with the oracle; 265 steps to 1e-4 (Table 1)."""
    s, val, b, _ = system("P1", None, 2)
    P = gsk.Plan(gsk.CSR(s["row_ptr"], s["col"], val), orth="cgs2")
    g = P.gmres(b, m=10, tol=1e-10, maxit=600)
    o = oracle.gmres(s["row_ptr"], s["col"], val, b, 10, 1e-10, 600, orth="cgs2")
    assert_same_solve(g, o)
    assert int(np.flatnonzero(g[1] < 1e-4)[0]) == 265


@pytest.mark.parametrize("engine", ["auto", "graph", "coop", "small", "cluster"])
def test_solver_edge_cases(engine):
    n = 300
    rp = np.arange(n + 1, dtype=np.int32)
    col = np.arange(n, dtype=np.int32)
    ones = np.ones(n)
    b = workloads.uniform(n, 1, 2)
    A = gsk.CSR(rp, col, ones)
    P = gsk.Plan(A, engine=engine)
    # A = I: Bi-CGSTAB half-step exit at iteration 1; GMRES 1 step (lucky)
    assert_same_solve(P.bicgstab(b, tol=1e-12, maxit=10), oracle.bicgstab(rp, col, ones, b, 1e-12, 10))
    Pf = gsk.Plan(A, schedule="fused", engine=engine)
    assert_same_solve(Pf.bicgstab(b, tol=1e-12, maxit=10), oracle.bicgstab(rp, col, ones, b, 1e-12, 10))
    assert_same_solve(P.gmres(b, m=5, tol=1e-12, maxit=10), oracle.gmres(rp, col, ones, b, 5, 1e-12, 10))
    # b = 0: converged at 0
    z = np.zeros(n)
    assert_same_solve(P.bicgstab(z, tol=1e-8, maxit=10), oracle.bicgstab(rp, col, ones, z, 1e-8, 10))
    assert_same_solve(P.gmres(z, m=5, tol=1e-8, maxit=10), oracle.gmres(rp, col, ones, z, 5, 1e-8, 10))
    # nonzero x0
    s = workloads.generate("C2", N=50)
    x0 = workloads.uniform(s["n"], 3, 4)
    P2 = gsk.Plan(gsk.CSR.from_system(s), engine=engine)
    assert_same_solve(P2.bicgstab(s["b"], x0=x0, tol=1e-9, maxit=300),
                      oracle.bicgstab(s["row_ptr"], s["col"], s["val"], s["b"], 1e-9, 300, x0=x0))
    assert_same_solve(P2.gmres(s["b"], x0=x0, m=7, tol=1e-9, maxit=300),
                      oracle.gmres(s["row_ptr"], s["col"], s["val"], s["b"], 7, 1e-9, 300, x0=x0))
    # breakdown: skew 2x2 gives <r0^, A r0> = 0 at iteration 1
    rp2 = np.array([0, 1, 2], np.int32)
    c2 = np.array([1, 0], np.int32)
    v2 = np.array([1.0, -1.0])
    bb = np.array([1.0, 0.0])
    for sched in ("fused", "split"):
        g = gsk.Plan(gsk.CSR(rp2, c2, v2), schedule=sched, engine=engine).bicgstab(bb, tol=1e-10, maxit=10)
        assert_same_solve(g, oracle.bicgstab(rp2, c2, v2, bb, 1e-10, 10))
        assert g[2]["status"] == 2 and g[2]["breakdown_at"] == 1
    # maxit = 1 and m >= n
    s3 = workloads.generate("C1", N=6)
    P3 = gsk.Plan(gsk.CSR.from_system(s3), engine=engine)
    assert_same_solve(P3.bicgstab(s3["b"], tol=1e-14, maxit=1),
                      oracle.bicgstab(s3["row_ptr"], s3["col"], s3["val"], s3["b"], 1e-14, 1))
    assert_same_solve(P3.gmres(s3["b"], m=40, tol=1e-14, maxit=100),
                      oracle.gmres(s3["row_ptr"], s3["col"], s3["val"], s3["b"], 40, 1e-14, 100))


VERDICTS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "verdict_systems.json")))["cases"]


def _csr_dense(A):
    rp, col, val = [0], [], []
    for row in A:
        nz = np.nonzero(row)[0]
        col += list(nz)
        val += list(row[nz])
        rp.append(len(col))
    return np.array(rp, np.int32), np.array(col, np.int32), np.array(val, np.float64)


@pytest.mark.parametrize("engine", ["auto", "graph", "coop", "small", "cluster"])
@pytest.mark.parametrize("case", VERDICTS, ids=[c["name"] for c in VERDICTS])
def test_verdict_branches(case, engine):
    """Every termination branch (readings B4/B5/B8) on the hand-derived
    systems of tests/golden/verdict_systems.json, on every engine and both Bi-CGSTAB
    schedules: GPU == oracle (NaN == NaN for DIVERGED) and the derived verdict."""
    if engine == "coop" and case["solver"] == "gmres":
        pytest.skip("the cooperative engine is Bi-CGSTAB only")
    A = np.array(case["A"], np.float64)
    b = np.array(case["b"], np.float64)
    rp, col, val = _csr_dense(A)
    e = case["expect"]
    for fmt in ("csr", "sell"):
        for schedule in (("split", "fused") if case["solver"] == "bicgstab" else ("split",)):
            P = gsk.Plan(gsk.CSR(rp, col, val), fmt=fmt, schedule=schedule, engine=engine)
            if case["solver"] == "bicgstab":
                g = P.bicgstab(b, tol=case["tol"], maxit=case["maxit"])
                o = oracle.bicgstab(rp, col, val, b, case["tol"], case["maxit"])
            else:
                g = P.gmres(b, m=case["m"], tol=case["tol"], maxit=case["maxit"])
                o = oracle.gmres(rp, col, val, b, case["m"], case["tol"], case["maxit"])
            assert_same_solve(g, o)
            assert (g[2]["status"], g[2]["iterations"], g[2]["breakdown_at"]) == \
                (e["status"], e["iterations"], e["breakdown_at"])
            P.close()


@pytest.mark.parametrize("weights", [False, True])
def test_problem1_unscaled_exact_breakdown(weights):
    """Problem 1 at 128^2 unscaled (PAPER.md:328-347, Table 1's "no conv.", :375):
    Bi-CGSTAB meets an exact-zero breakdown test (B5) at iteration 913 — GPU ==
    oracle through the breakdown, stopping in the solved or the GS(2) frame."""
    s = workloads.generate("P1")
    w = oracle.gs_scale(s["row_ptr"], s["val"], s["b"], 2)[2] if weights else None
    P = gsk.Plan(gsk.CSR.from_system(s), fmt="sell", weights=w)
    g = P.bicgstab(s["b"], tol=1e-10, maxit=10000)
    o = oracle.bicgstab(s["row_ptr"], s["col"], s["val"], s["b"], 1e-10, 10000, weights=w)
    assert_same_solve(g, o)
    assert g[2]["status"] == 2 and g[2]["breakdown_at"] == 913


SMALL = [("C1", None), ("C1", 20), ("C2", 40), ("C2", 64), ("C3", 12), ("C3", 16), ("C4", 10), ("C5", 50),
         ("P1", 64)]


@pytest.mark.parametrize("name,N", SMALL)
@pytest.mark.parametrize("scaling", ["none", 2])
def test_small_engine_parity(name, N, scaling):
    """The on-chip single-CTA solvers (small.cu; n <= 4096, ragged n included) against
    the oracle and against the graph-replayed passes: Bi-CGSTAB (both schedules, SELL
    and CSR plans, frame weights) and GMRES(m) with MGS for m in {1, 20, 30}."""
    s, val, b, _ = system(name, N, scaling)
    assert s["n"] <= 4096
    A = gsk.CSR(s["row_ptr"], s["col"], val)
    o = oracle.bicgstab(s["row_ptr"], s["col"], val, b, 1e-9, 800)
    for fmt in ("csr", "sell"):
        for schedule in ("split", "fused"):
            P = gsk.Plan(A, fmt=fmt, schedule=schedule, engine="small")
            assert_same_solve(P.bicgstab(b, tol=1e-9, maxit=800), o)
    assert_same_solve(gsk.Plan(A, engine="graph").bicgstab(b, tol=1e-9, maxit=800), o)
    w = workloads.uniform(s["n"], 5, 6) + 1.5
    assert_same_solve(gsk.Plan(A, weights=w, engine="small").bicgstab(b, tol=1e-9, maxit=800),
                      oracle.bicgstab(s["row_ptr"], s["col"], val, b, 1e-9, 800, weights=w))
    for m in (1, 20, 30):
        o = oracle.gmres(s["row_ptr"], s["col"], val, b, m, 1e-9, 300)
        assert_same_solve(gsk.Plan(A, engine="small").gmres(b, m=m, tol=1e-9, maxit=300), o)
        if m == 20:
            assert_same_solve(gsk.Plan(A, engine="graph").gmres(b, m=m, tol=1e-9, maxit=300), o)
            assert_same_solve(gsk.Plan(A, fmt="sell").gmres(b, m=m, tol=1e-9, maxit=300), o)
            assert_same_solve(gsk.Plan(A, weights=w).gmres(b, m=m, tol=1e-9, maxit=300),
                              oracle.gmres(s["row_ptr"], s["col"], val, b, m, 1e-9, 300, weights=w))


def test_plan_less_entry_points():
    s = workloads.generate("C1")
    A = gsk.CSR.from_system(s)
    assert_same_solve(gsk.bicgstab_solve(A, s["b"], tol=1e-8, maxit=300),
                      oracle.bicgstab(s["row_ptr"], s["col"], s["val"], s["b"], 1e-8, 300))
    assert_same_solve(gsk.gmres_solve(A, s["b"], m=20, tol=1e-8, maxit=300),
                      oracle.gmres(s["row_ptr"], s["col"], s["val"], s["b"], 20, 1e-8, 300))


def test_repeat_solves_are_deterministic():
    s = workloads.generate("C3", N=16)
    P = gsk.Plan(gsk.CSR.from_system(s), fmt="sell", engine="graph")
    a = P.bicgstab(s["b"], tol=1e-9, maxit=500)
    b = P.bicgstab(s["b"], tol=1e-9, maxit=500)
    assert np.array_equal(a[1], b[1]) and np.array_equal(cpu(a[0]), cpu(b[0]))
    c = P.gmres(s["b"], m=30, tol=1e-9, maxit=300)
    d = P.gmres(s["b"], m=30, tol=1e-9, maxit=300)
    assert np.array_equal(c[1], d[1]) and np.array_equal(cpu(c[0]), cpu(d[0]))


# ---------------------------------------------------------------- full BASELINE sizes
@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_full_size_parity(name):
    """Each BASELINE config at full size, in the launch configuration bench.py uses
    (GS(2) then SELL for C4, CSR otherwise): GS bit-exact, the first 50 Bi-CGSTAB
    iterations and one GMRES(30) cycle + 2 steps bit-exact against the oracle."""
    c = workloads.CONFIGS[name]
    s = workloads.generate(name)
    A = gsk.CSR.from_system(s)
    As, bs, d = gsk.gs_scale(A, s["b"], 2)
    vo, bo, do = oracle.gs_scale(s["row_ptr"], s["val"], s["b"], 2)
    assert np.array_equal(cpu(As.val), vo) and np.array_equal(cpu(bs), bo)
    P = gsk.Plan(As, fmt="sell" if c.sell else "csr")
    g = P.bicgstab(bs, tol=c.tol, maxit=50)
    o = oracle.bicgstab(s["row_ptr"], s["col"], vo, bo, c.tol, 50)
    assert_same_solve(g, o)
    g = P.gmres(bs, m=30, tol=c.tol, maxit=32)
    o = oracle.gmres(s["row_ptr"], s["col"], vo, bo, 30, c.tol, 32)
    assert_same_solve(g, o)
    if name in ("C2", "C4"):
        Pc = gsk.Plan(As, fmt="sell" if c.sell else "csr", orth="cgs2")
        g = Pc.gmres(bs, m=30, tol=c.tol, maxit=32)
        o = oracle.gmres(s["row_ptr"], s["col"], vo, bo, 30, c.tol, 32, orth="cgs2")
        assert_same_solve(g, o)


@pytest.mark.parametrize("name,N", [("C1", None), ("C3", 20), ("C4", 24), ("C5", 96), ("P1", 64)])
@pytest.mark.parametrize("p", [1, 2])
def test_two_sided_scaling_parity(name, N, p):
    """D^1/2 A D^1/2: scaled values, b, s bit-exact; a Bi-CGSTAB solve
    of the scaled system and the unscaled x bit-exact."""
    s = workloads.generate(name, N=N)
    A = gsk.CSR.from_system(s)
    As, bs, sv = gsk.gs_scale_sym(A, s["b"], p)
    vo, bo, so = oracle.gs_scale_sym(s["row_ptr"], s["col"], s["val"], s["b"], p)
    assert np.array_equal(cpu(As.val), vo) and np.array_equal(cpu(bs), bo) and np.array_equal(cpu(sv), so)
    g = gsk.Plan(As).bicgstab(bs, tol=1e-9, maxit=500)
    o = oracle.bicgstab(s["row_ptr"], s["col"], vo, bo, 1e-9, 500)
    assert_same_solve(g, o)
    assert np.array_equal(cpu(gsk.gs_unscale(sv, g[0])), oracle.unscale(so, o[0]))


# ---------------------------------------------------------------- row-block shards (f4)
SHARDED = [("C1", None, 2), ("C1", None, 8), ("C2", 64, 4), ("C3", 16, 4), ("C4", 24, 2), ("C4", 24, 4),
           ("C5", 64, 2), ("P1", 64, 8)]


@pytest.mark.parametrize("name,N,P", SHARDED)
def test_sharded_parity(name, N, P):
    """All P shards on this GPU (halo exchange by device copies, shard values gathered
    and joined by the top of the canonical tree): Bi-CGSTAB and MGS
    GMRES bit-identical to the oracle, CSR and SELL shards, weights and x0."""
    s, val, b, _ = system(name, N, 2)
    A = gsk.CSR(s["row_ptr"], s["col"], val)
    ob = oracle.bicgstab(s["row_ptr"], s["col"], val, b, 1e-9, 500)
    og = oracle.gmres(s["row_ptr"], s["col"], val, b, 20, 1e-9, 200)
    for fmt in ("csr", "sell"):
        SP = gsk.ShardedPlan(A, shards=P, fmt=fmt)
        assert_same_solve(SP.bicgstab(b, tol=1e-9, maxit=500), ob)
        assert_same_solve(SP.gmres(b, m=20, tol=1e-9, maxit=200), og)
        SP.close()
    w = workloads.uniform(s["n"], 5, 6) + 1.5
    x0 = workloads.uniform(s["n"], 7, 8)
    SP = gsk.ShardedPlan(A, shards=P, weights=w)
    assert_same_solve(SP.bicgstab(b, x0=x0, tol=1e-9, maxit=500),
                      oracle.bicgstab(s["row_ptr"], s["col"], val, b, 1e-9, 500, x0=x0, weights=w))
    assert_same_solve(SP.gmres(b, x0=x0, m=7, tol=1e-9, maxit=200),
                      oracle.gmres(s["row_ptr"], s["col"], val, b, 7, 1e-9, 200, x0=x0, weights=w))


def test_sharded_rejections():
    s = workloads.generate("C5", N=64)
    with pytest.raises(gsk.GskError):  # permuted: halos beyond the adjacent shards
        gsk.ShardedPlan(gsk.CSR.from_system(s), shards=8)
    s = workloads.generate("C1")
    SP = gsk.ShardedPlan(gsk.CSR.from_system(s), shards=2)
    SP.close()
    with pytest.raises(gsk.GskError):
        gsk.ShardedPlan(gsk.CSR.from_system(s), shards=3)


def test_sharded_full_c4_matches_unsharded():
    """C4 at full size in 8 SELL shards on one GPU: the first 30 Bi-CGSTAB iterations
    and 35 GMRES(30) steps are bit-identical to the unsharded plan (itself bit-exact
    with the oracle, test_full_size_parity)."""
    s = workloads.generate("C4")
    A0 = gsk.CSR.from_system(s)
    As, bs, _ = gsk.gs_scale(A0, s["b"], 2)
    P1 = gsk.Plan(As, fmt="sell")
    g1 = P1.bicgstab(bs, tol=1e-8, maxit=30)
    h1 = P1.gmres(bs, m=30, tol=1e-8, maxit=35)
    P1.close()
    SP = gsk.ShardedPlan(As, shards=8, fmt="sell")
    g8 = SP.bicgstab(bs, tol=1e-8, maxit=30)
    h8 = SP.gmres(bs, m=30, tol=1e-8, maxit=35)
    for a, c in ((g1, g8), (h1, h8)):
        assert np.array_equal(a[1], c[1])
        assert torch.equal(a[0], c[0])
        for k in ("status", "iterations", "relres", "true_relres"):
            assert a[2][k] == c[2][k]


def test_nccl_plumbing_single_rank():
    """The NCCL entry points the multi-process shards use (libnccl.so.2 loaded at run
    time next to torch's): unique id, a 1-rank communicator, destroy."""
    import ctypes
    lib = gsk.load()
    buf = ctypes.create_string_buffer(128)
    assert lib.gsk_nccl_unique_id(buf) == 0
    h = ctypes.c_void_p()
    assert lib.gsk_nccl_comm_create(ctypes.c_char_p(bytes(buf.raw)), 1, 0, ctypes.byref(h)) == 0
    assert h.value
    assert lib.gsk_nccl_comm_destroy(h) == 0


def test_bench_sharded_line():
    """bench.py --shards (emulated on one GPU): one JSON line, the sharded solve converges
    with the unsharded iteration count."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, GSK_BENCH_NO_CLOCKS="1")
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--config", "C3", "--N", "32",
                          "--shards", "4", "--steps", "1", "--warmup", "1"], capture_output=True, text=True,
                         check=True, timeout=600, env=env).stdout
    line = json.loads(out.strip().splitlines()[-1])
    assert line["config"]["shards"] == 4 and line["value"] > 0 and line["gpu_launches"] > 0
    s = workloads.generate("C3", N=32)
    _, vo, bo, _ = system("C3", 32, 2)
    o = oracle.bicgstab(s["row_ptr"], s["col"], vo, bo, workloads.CONFIGS["C3"].tol, 10000)
    assert line["extra"]["bicgstab"]["iterations"] == o[2]["iterations"]


@pytest.mark.parametrize("name,N,P", [("C3", 16, 4), ("C4", 24, 2), ("C1", None, 8)])
def test_sharded_spmv(name, N, P):
    s = workloads.generate(name, N=N)
    x = workloads.uniform(s["n"], 9, 9)
    y = oracle.spmv(s["row_ptr"], s["col"], s["val"], x)
    for fmt in ("csr", "sell"):
        SP = gsk.ShardedPlan(gsk.CSR.from_system(s), shards=P, fmt=fmt)
        assert np.array_equal(cpu(SP.spmv(x)), y)
        SP.close()


def test_solver_argument_errors():
    """API errors are negative returns with a message (include/gsk.h), never a crash:
    tol <= 0, maxit < 1, m out of range, CGS2 beyond its m limit, unknown options; a
    failed call leaves the plan usable."""
    s = workloads.generate("C2", N=40)
    A = gsk.CSR.from_system(s)
    P = gsk.Plan(A)
    bad = [lambda: P.bicgstab(s["b"], tol=0.0), lambda: P.bicgstab(s["b"], maxit=0),
           lambda: P.gmres(s["b"], m=0), lambda: P.gmres(s["b"], m=129), lambda: P.gmres(s["b"], tol=-1.0),
           lambda: gsk.Plan(A, orth="cgs2", engine="graph").gmres(s["b"], m=65, maxit=10)]
    for f in bad:
        with pytest.raises(gsk.GskError) as ei:
            f()
        assert ei.value.code == -1 and str(ei.value)
    for kw in ({"fmt": "dia"}, {"schedule": "x"}, {"orth": "x"}, {"engine": "x"}):
        with pytest.raises(KeyError):
            gsk.Plan(A, **kw)
    assert_same_solve(P.bicgstab(s["b"], tol=1e-9, maxit=300),
                      oracle.bicgstab(s["row_ptr"], s["col"], s["val"], s["b"], 1e-9, 300))


CLUSTER = [("C1", None), ("C2", 50), ("C3", 16), ("C5", 96), ("P1", None), ("C4", 24), ("C3", 32), ("C2", 200),
           ("P4conv", None)]


@pytest.mark.parametrize("name,N", CLUSTER)
def test_cluster_engine_parity(name, N):
    """On-chip solvers on one thread-block cluster (cluster.cu; up to 16 CTAs with DSMEM
    reductions, n <= 16384, ragged n included): Bi-CGSTAB and MGS GMRES bit-exact
    against the oracle, with and without frame weights."""
    s, val, b, _ = system(name, N, 2)
    if s["n"] > 65536:
        pytest.skip("beyond one cluster")
    A = gsk.CSR(s["row_ptr"], s["col"], val)
    P = gsk.Plan(A, engine="cluster")
    assert_same_solve(P.bicgstab(b, tol=1e-9, maxit=600), oracle.bicgstab(s["row_ptr"], s["col"], val, b, 1e-9, 600))
    for m in (1, 20, 30):
        assert_same_solve(P.gmres(b, m=m, tol=1e-9, maxit=200),
                          oracle.gmres(s["row_ptr"], s["col"], val, b, m, 1e-9, 200))
    w = workloads.uniform(s["n"], 5, 6) + 1.5
    Pw = gsk.Plan(A, engine="cluster", weights=w)
    assert_same_solve(Pw.bicgstab(b, tol=1e-9, maxit=600),
                      oracle.bicgstab(s["row_ptr"], s["col"], val, b, 1e-9, 600, weights=w))
    assert_same_solve(Pw.gmres(b, m=20, tol=1e-9, maxit=200),
                      oracle.gmres(s["row_ptr"], s["col"], val, b, 20, 1e-9, 200, weights=w))


COOP = [("C2", 128, None), ("C2", 264, None), ("C2", 200, "7"), ("C5", 200, None), ("C3", 32, "5"),
        ("C2", 264, "1"), ("C4", 24, None)]


@pytest.mark.parametrize("name,N,gcap", COOP)
@pytest.mark.parametrize("fmt", ["csr", "sell"])
def test_coop_engine_parity(name, N, gcap, fmt, monkeypatch):
    """Persistent cooperative Bi-CGSTAB (coop.cu: per-CTA epoch flags, every CTA
    reducing the CTA partials itself): bit-exact against the oracle over grids of one
    CTA, of G > 256 CTAs (two partials per finish thread) and of capped grids with
    several windows per CTA (GSK_COOP_G), natural / sorted SELL windows and CSR, with
    and without frame weights."""
    if gcap:
        monkeypatch.setenv("GSK_COOP_G", gcap)
    s, val, b, _ = system(name, N, 2)
    A = gsk.CSR(s["row_ptr"], s["col"], val)
    P = gsk.Plan(A, fmt=fmt, engine="coop")
    assert_same_solve(P.bicgstab(b, tol=1e-10, maxit=400),
                      oracle.bicgstab(s["row_ptr"], s["col"], val, b, 1e-10, 400))
    w = workloads.uniform(s["n"], 5, 6) + 1.5
    Pw = gsk.Plan(A, fmt=fmt, engine="coop", weights=w)
    assert_same_solve(Pw.bicgstab(b, tol=1e-10, maxit=300),
                      oracle.bicgstab(s["row_ptr"], s["col"], val, b, 1e-10, 300, weights=w))


def test_concurrent_plans_two_threads():
    """Two plans driven from two host threads at once (each on its own stream, the GIL
    released inside the C calls): both solves stay bit-exact."""
    import threading
    jobs = [("C2", 64, "graph"), ("C3", 20, "graph"), ("C4", 24, "auto"), ("P1", 64, "auto")]
    res = {}

    errors = []

    def work(name, N, engine):
        try:
            s, val, b, _ = system(name, N, 2)
            P = gsk.Plan(gsk.CSR(s["row_ptr"], s["col"], val), engine=engine)
            for _ in range(3):
                g = P.bicgstab(b, tol=1e-9, maxit=400)
                h = P.gmres(b, m=20, tol=1e-9, maxit=100)
            # a stream-level sync: a device-wide one would invalidate the other threads'
            # graph captures (the library retries a failed capture)
            torch.cuda.current_stream().synchronize()
            res[name] = (s, val, b, g, h)
        except Exception as e:  # noqa: BLE001 (reported below)
            errors.append((name, repr(e)))

    threads = [threading.Thread(target=work, args=j) for j in jobs]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors and len(res) == len(jobs), errors
    for name, (s, val, b, g, h) in res.items():
        assert_same_solve(g, oracle.bicgstab(s["row_ptr"], s["col"], val, b, 1e-9, 400))
        assert_same_solve(h, oracle.gmres(s["row_ptr"], s["col"], val, b, 20, 1e-9, 100))


def test_capture_survives_device_syncs_from_another_thread():
    """A host thread calling cudaDeviceSynchronize while another thread's plan captures
    its graphs invalidates that capture; the library retries it, so the solve still
    returns the oracle's bits (the syncing thread may see the CUDA error; it is
    ignored here)."""
    import threading
    s, val, b, _ = system("C3", 20, 2)
    stop = threading.Event()

    def hammer():
        while not stop.is_set():
            try:
                torch.cuda.synchronize()
            except Exception:  # noqa: BLE001 (cudaErrorStreamCaptureUnsupported: expected)
                pass
            stop.wait(0.005)

    th = threading.Thread(target=hammer)
    th.start()
    try:
        for _ in range(3):
            P = gsk.Plan(gsk.CSR(s["row_ptr"], s["col"], val), engine="graph", fmt="sell")
            assert_same_solve(P.bicgstab(b, tol=1e-9, maxit=400),
                              oracle.bicgstab(s["row_ptr"], s["col"], val, b, 1e-9, 400))
            P.close()
    finally:
        stop.set()
        th.join()


@pytest.mark.parametrize("name,N", [("C4", 24), ("C3", 20), ("C2", 100)])
def test_sell_dict_solvers(name, N):
    """Solvers on SELL-D plans (uint8 column index into per-chunk deltas): the same bits."""
    s, val, b, _ = system(name, N, 2)
    P = gsk.Plan(gsk.CSR(s["row_ptr"], s["col"], val), fmt="sell", sell_index="dict", engine="graph")
    assert P.sell_dict() is not None
    assert_same_solve(P.bicgstab(b, tol=1e-9, maxit=400), oracle.bicgstab(s["row_ptr"], s["col"], val, b, 1e-9, 400))
    assert_same_solve(P.gmres(b, m=30, tol=1e-9, maxit=100),
                      oracle.gmres(s["row_ptr"], s["col"], val, b, 30, 1e-9, 100))


@pytest.mark.parametrize("kind,k", [("rho0", 7), ("omega0", 7), ("nan", 7), ("nan", 1)])
@pytest.mark.parametrize("fmt,schedule", [("csr", "split"), ("sell", "split"), ("sell", "fused"), ("sell", "split4")])
def test_fault_hook_parity(kind, k, fmt, schedule, monkeypatch):
    """The test-only fault hook on both sides — GSK_FAULT on the GPU,
    oracle.set_fault on the host — reaches the breakdown and divergence verdicts on a
    system that has none, with identical iterates, history and verdict."""
    s, val, b, _ = system("C3", 20, 2)
    A = gsk.CSR(s["row_ptr"], s["col"], val)
    P = gsk.Plan(A, fmt=fmt, schedule=schedule, engine="graph")
    monkeypatch.setenv("GSK_FAULT", f"{kind}:{k}")
    try:
        oracle.set_fault(kind, k)
        o = oracle.bicgstab(s["row_ptr"], s["col"], val, b, 1e-9, 400)
    finally:
        oracle.set_fault()
    g = P.bicgstab(b, tol=1e-9, maxit=400)
    assert o[2]["status"] == (3 if kind == "nan" else 2)
    assert_same_solve(g, o)


@pytest.mark.parametrize("name,N", [("C1", None), ("C2", 100), ("C3", 20), ("C4", 24), ("C4", None), ("C5", 64),
                                    ("P4", 12)])
def test_sell_uniform_parity(name, N):
    """SELL-U (chunk-uniform column deltas) built on the device == the oracle's encoding
    (integer arrays and values bit-exact; also after a value refresh); the permuted C5
    system keeps plain int32 columns on both sides."""
    s = workloads.generate(name, N=N)
    A = gsk.CSR.from_system(s)
    P = gsk.Plan(A, fmt="sell", sell_index="uniform")
    g = P.sell_uniform()
    o = oracle.sell_uniform(s["row_ptr"], s["col"], s["val"], oracle.sell_build(s["row_ptr"], s["col"], s["val"]))
    if o is None:
        assert g is None
        return
    for k in ("uptr", "udel", "umask", "uval"):
        assert np.array_equal(g[k], o[k]), k
    vo, _, _ = oracle.gs_scale(s["row_ptr"], s["val"], s["b"], 2)  # refresh after rescaling in place
    A.val.copy_(torch.tensor(vo, device="cuda"))
    P.refresh()
    o2 = oracle.sell_uniform(s["row_ptr"], s["col"], vo, oracle.sell_build(s["row_ptr"], s["col"], vo))
    assert np.array_equal(P.sell_uniform()["uval"], o2["uval"])
    x = workloads.uniform(s["n"], 9, 9)
    assert np.array_equal(cpu(P.spmv(x)), oracle.spmv(s["row_ptr"], s["col"], vo, x))


@pytest.mark.parametrize("name,N", [("C4", 24), ("C3", 20), ("C2", 100), ("P1", 64)])
def test_sell_uniform_solvers(name, N):
    """Solvers on SELL-U plans (no per-slot column data): the same bits as the oracle —
    split and fused Bi-CGSTAB, MGS and CGS2 GMRES, with frame weights, and sharded."""
    s, val, b, _ = system(name, N, 2)
    A = gsk.CSR(s["row_ptr"], s["col"], val)
    ob = oracle.bicgstab(s["row_ptr"], s["col"], val, b, 1e-9, 400)
    og = oracle.gmres(s["row_ptr"], s["col"], val, b, 30, 1e-9, 100)
    for schedule in ("split", "fused"):
        P = gsk.Plan(A, fmt="sell", sell_index="uniform", engine="graph", schedule=schedule)
        assert P.sell_uniform() is not None
        assert_same_solve(P.bicgstab(b, tol=1e-9, maxit=400), ob)
        assert_same_solve(P.gmres(b, m=30, tol=1e-9, maxit=100), og)
    P = gsk.Plan(A, fmt="sell", sell_index="uniform", engine="graph", orth="cgs2")
    assert_same_solve(P.gmres(b, m=30, tol=1e-9, maxit=100),
                      oracle.gmres(s["row_ptr"], s["col"], val, b, 30, 1e-9, 100, orth="cgs2"))
    w = workloads.uniform(s["n"], 5, 6) + 1.5
    Pw = gsk.Plan(A, fmt="sell", sell_index="uniform", engine="graph", weights=w)
    assert_same_solve(Pw.bicgstab(b, tol=1e-9, maxit=400),
                      oracle.bicgstab(s["row_ptr"], s["col"], val, b, 1e-9, 400, weights=w))
    SP = gsk.ShardedPlan(A, shards=2, fmt="sell", sell_index="uniform")
    assert_same_solve(SP.bicgstab(b, tol=1e-9, maxit=400), ob)
    assert_same_solve(SP.gmres(b, m=30, tol=1e-9, maxit=100), og)


@pytest.mark.parametrize("name,N", [("C1", None), ("C2", 100), ("C3", 20), ("C3", 48), ("C4", 24), ("C4", 64),
                                    ("C5", 64), ("P4", 12), ("P1", 64)])
def test_row_classes_parity(name, N):
    """Row-class dictionary (RCD) built on the device == the oracle's encoding: class ids
    (first-occurrence numbering), lengths, deltas and values bit for bit — also after a
    value refresh (GS(2) in place) — and the plan's SpMV == the oracle's; systems whose
    rows do not repeat (C2's node-dependent velocity at size, permuted C5) are inapplicable
    on both sides and keep their SELL passes."""
    s = workloads.generate(name, N=N)
    A = gsk.CSR.from_system(s)
    P = gsk.Plan(A, fmt="sell", sell_index="classes")
    x = workloads.uniform(s["n"], 9, 9)
    for val in (s["val"], oracle.gs_scale(s["row_ptr"], s["val"], s["b"], 2)[0]):
        if val is not s["val"]:
            A.val.copy_(torch.tensor(val, device="cuda"))
            P.refresh()
        g = P.row_classes()
        o = oracle.row_classes(s["row_ptr"], s["col"], val)
        assert (g is None) == (o is None)
        if o is not None:
            for k in ("cls", "len", "delta"):
                assert np.array_equal(g[k], o[k]), k
            assert np.array_equal(g["val"].view(np.uint64), o["val"].view(np.uint64))
        assert np.array_equal(cpu(P.spmv(x)), oracle.spmv(s["row_ptr"], s["col"], val, x))


def _banded_system(n, deltas, seed):
    """Rows with entries at the given deltas (inside [0, n)), values from a few repeating
    patterns (so the rows fall into classes), diagonally dominant."""
    pat = np.array([[-1.0, 4.5, -0.5, -1.25], [-2.0, 7.0, -1.5, -0.75], [0.5, 3.0, -0.25, 1.0]])
    rp, cols, vals = [0], [], []
    for r in range(n):
        k = (r // 97) % 3
        for d, v in zip(deltas, pat[k]):
            if 0 <= r + d < n:
                cols.append(r + d)
                vals.append(v)
        rp.append(len(cols))
    b = workloads.uniform(n, seed, 1)
    return np.array(rp, np.int32), np.array(cols, np.int32), np.array(vals), b


def test_row_classes_with_empty_rows():
    """Empty rows form a class of length 0 (y = +0.0 there, as in CSR); the other rows of
    these 5- / 7-point Laplacians keep the plan's stencil slots."""
    for name, N in (("lap2d", 40), ("lap3d", 12)):
        s = workloads.generate(name, N=N)
        rp, col, val = s["row_ptr"], s["col"], s["val"]
        keep = np.ones(len(col), bool)
        for r in range(3, s["n"], 37):
            keep[rp[r]:rp[r + 1]] = False
        ln = np.add.reduceat(keep.astype(np.int64), rp[:-1])
        rp2 = np.concatenate([[0], np.cumsum(ln)]).astype(np.int32)
        col2, val2 = col[keep], val[keep]
        A = gsk.CSR(rp2, col2, val2)
        P = gsk.Plan(A, fmt="sell", sell_index="classes", engine="graph")
        o = oracle.row_classes(rp2, col2, val2)
        g = P.row_classes()
        assert g is not None and np.array_equal(g["cls"], o["cls"]) and 0 in list(o["len"])
        x = workloads.uniform(s["n"], 9, 9)
        y = cpu(P.spmv(x))
        assert np.array_equal(y, oracle.spmv(rp2, col2, val2, x))
        assert not np.signbit(y[3]) and y[3] == 0.0


def test_row_classes_without_stencil_slots():
    """Classes whose deltas are no symmetric 5- / 7-point set (here {-3, 0, 1, 7}) run the
    generic class-line kernels (no stencil slots): SpMV and both solvers == the oracle."""
    rp, col, val, b = _banded_system(5000, (-3, 0, 1, 7), 5)
    A = gsk.CSR(rp, col, val)
    P = gsk.Plan(A, fmt="sell", sell_index="classes", engine="graph")
    assert P.row_classes() is not None and P.class_slots() is None
    x = workloads.uniform(5000, 9, 9)
    assert np.array_equal(cpu(P.spmv(x)), oracle.spmv(rp, col, val, x))
    assert_same_solve(P.bicgstab(b, tol=1e-10, maxit=200), oracle.bicgstab(rp, col, val, b, 1e-10, 200))
    assert_same_solve(P.gmres(b, m=20, tol=1e-10, maxit=100), oracle.gmres(rp, col, val, b, 20, 1e-10, 100))


@pytest.mark.parametrize("name,N,ns,roll", [("C4", 24, 7, False), ("C3", 20, 7, False), ("P1", 64, 5, False),
                                            ("C1", 256, 5, True), ("C1", None, 5, False), ("P4", 12, 7, False)])
def test_class_slots_parity(name, N, ns, roll):
    """Stencil slots of a row-class plan: the plan's delta set is the union of the oracle
    classes' deltas (symmetric, 5 or 7), every class's mask and values decode back to the
    oracle's class line (ascending delta = CSR order), and the passes on them — with the
    +-256 entries taken from the thread's neighbouring windows when a grid line is one
    window (P1 at 256^2) — give the oracle's bits."""
    s, val, b, _ = system(name, N, 2)
    A = gsk.CSR(s["row_ptr"], s["col"], val)
    P = gsk.Plan(A, fmt="sell", sell_index="classes", engine="graph")
    S = P.class_slots()
    o = oracle.row_classes(s["row_ptr"], s["col"], val)
    assert S is not None and len(S["deltas"]) == ns
    U = sorted({int(d) for k, L in enumerate(o["len"]) for d in o["delta"][k, :L]})
    assert list(S["deltas"]) == U and (U[ns // 2 + 2] == 256) == roll
    for k, L in enumerate(o["len"]):
        pos = [U.index(int(d)) for d in o["delta"][k, :L]]
        assert int(S["mask"][k]) == sum(1 << q for q in pos)
        assert np.array_equal(S["val"][k, pos].view(np.uint64), o["val"][k, :L].view(np.uint64))
        assert not S["val"][k, [q for q in range(8) if q not in pos]].any()
    x = workloads.uniform(s["n"], 9, 9)
    assert np.array_equal(cpu(P.spmv(x)), oracle.spmv(s["row_ptr"], s["col"], val, x))
    assert_same_solve(P.bicgstab(b, tol=1e-9, maxit=120), oracle.bicgstab(s["row_ptr"], s["col"], val, b, 1e-9, 120))
    assert_same_solve(P.gmres(b, m=30, tol=1e-9, maxit=60), oracle.gmres(s["row_ptr"], s["col"], val, b, 30, 1e-9, 60))


def test_row_classes_hash_collision_falls_back():
    """Lossless by construction: with the hash truncated to 3 bits (test hook
    GSK_RCD_HASH_BITS, read at the first build: a fresh process) different rows share a
    key, the entry-by-entry comparison with the class's first row catches it, and the plan
    keeps its SELL slot passes — the SpMV and Bi-CGSTAB still give the oracle's bits."""
    import subprocess
    import sys
    code = """
import numpy as np, oracle, workloads, paper_0812_2769_b200 as gsk
s = workloads.generate("C4", N=24)
val, b, _ = oracle.gs_scale(s["row_ptr"], s["val"], s["b"], 2)
A = gsk.CSR(s["row_ptr"], s["col"], val)
P = gsk.Plan(A, fmt="sell", sell_index="classes", engine="graph")
assert oracle.row_classes(s["row_ptr"], s["col"], val) is not None
assert P.row_classes() is None and P.num_classes() == -1, "collisions must make the format inapplicable"
x = workloads.uniform(s["n"], 9, 9)
assert np.array_equal(P.spmv(x).cpu().numpy(), oracle.spmv(s["row_ptr"], s["col"], val, x))
xg, hg, rg = P.bicgstab(b, tol=1e-9, maxit=60)
xo, ho, ro = oracle.bicgstab(s["row_ptr"], s["col"], val, b, 1e-9, 60)
assert np.array_equal(hg, ho) and np.array_equal(xg.cpu().numpy(), xo)
print("fallback ok")
"""
    env = dict(os.environ, GSK_RCD_HASH_BITS="3")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env["PYTHONPATH"] = root + os.pathsep + env.get("PYTHONPATH", "")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "fallback ok" in r.stdout, r.stdout + r.stderr


def test_row_classes_applicability_flips_on_refresh():
    """A refresh that makes the rows distinct (a value per row) drops the plan back to its
    SELL passes, and one that restores repeating rows brings the classes back; the solver
    graphs are re-captured each time (same bits as the oracle throughout)."""
    s, val, b, _ = system("C4", 24, 2)
    A = gsk.CSR(s["row_ptr"], s["col"], val.copy())
    P = gsk.Plan(A, fmt="sell", sell_index="classes", engine="graph")
    assert P.row_classes() is not None
    o = oracle.bicgstab(s["row_ptr"], s["col"], val, b, 1e-9, 60)
    assert_same_solve(P.bicgstab(b, tol=1e-9, maxit=60), o)
    v2 = val * (1.0 + 1e-3 * workloads.uniform(val.size, 3, 3))  # every row different
    A.val.copy_(torch.tensor(v2, device="cuda"))
    P.refresh()
    assert P.row_classes() is None
    assert_same_solve(P.bicgstab(b, tol=1e-9, maxit=60), oracle.bicgstab(s["row_ptr"], s["col"], v2, b, 1e-9, 60))
    A.val.copy_(torch.tensor(val, device="cuda"))
    P.refresh()
    assert P.row_classes() is not None
    assert_same_solve(P.bicgstab(b, tol=1e-9, maxit=60), o)


@pytest.mark.parametrize("name,N,scal", [("C4", 24, 2), ("C4", 40, 2), ("C3", 20, 2), ("C3", 33, 1), ("P1", 64, 2),
                                         ("C1", None, 2), ("P4", 12, "none")])
def test_row_classes_solvers(name, N, scal):
    """Solvers on row-class plans (no slot data read by the passes): the same bits as the
    oracle — split, four-pass and fused Bi-CGSTAB, MGS and CGS2 GMRES, frame weights, x0,
    and sharded (ragged sizes included: 33^3 and 40^3 rows are no multiple of 256)."""
    s, val, b, _ = system(name, N, scal)
    A = gsk.CSR(s["row_ptr"], s["col"], val)
    ob = oracle.bicgstab(s["row_ptr"], s["col"], val, b, 1e-9, 300)
    og = oracle.gmres(s["row_ptr"], s["col"], val, b, 30, 1e-9, 90)
    for schedule in ("split", "split4", "fused"):
        P = gsk.Plan(A, fmt="sell", sell_index="classes", engine="graph", schedule=schedule)
        assert P.row_classes() is not None
        assert_same_solve(P.bicgstab(b, tol=1e-9, maxit=300), ob)
        assert_same_solve(P.gmres(b, m=30, tol=1e-9, maxit=90), og)
    P = gsk.Plan(A, fmt="sell", sell_index="classes", engine="graph", orth="cgs2")
    assert_same_solve(P.gmres(b, m=30, tol=1e-9, maxit=90),
                      oracle.gmres(s["row_ptr"], s["col"], val, b, 30, 1e-9, 90, orth="cgs2"))
    w = workloads.uniform(s["n"], 5, 6) + 1.5
    x0 = workloads.uniform(s["n"], 7, 8)
    Pw = gsk.Plan(A, fmt="sell", sell_index="classes", engine="graph", weights=w)
    assert_same_solve(Pw.bicgstab(b, x0=x0, tol=1e-9, maxit=300),
                      oracle.bicgstab(s["row_ptr"], s["col"], val, b, 1e-9, 300, x0=x0, weights=w))
    # the default engine choice (on-chip / cooperative engines read the SELL slots)
    Pa = gsk.Plan(A, fmt="sell", sell_index="classes")
    assert_same_solve(Pa.bicgstab(b, tol=1e-9, maxit=300), ob)
    assert_same_solve(Pa.gmres(b, m=30, tol=1e-9, maxit=90), og)
    if s["n"] >= 4096:
        SP = gsk.ShardedPlan(A, shards=2, fmt="sell", sell_index="classes")
        assert_same_solve(SP.bicgstab(b, tol=1e-9, maxit=300), ob)
        assert_same_solve(SP.gmres(b, m=30, tol=1e-9, maxit=90), og)


@pytest.mark.parametrize("name,N,scal,m,tol", [("C1", None, 1, 20, 1e-4), ("C1", None, "none", 20, 1e-3),
                                               ("C3", 20, 1, 30, 1e-6), ("C4", 24, "none", 30, 1e-5),
                                               ("C2", 100, 1, 30, 1e-6), ("C4", 40, 2, 10, 1e-7)])
def test_gmres_weighted_stop_parity(name, N, scal, m, tol):
    """gsk_opts.gmres_wstop (reading B2w): GMRES stopping on the GS(2)-frame
    true residual at cycle ends == the oracle's orc_gmres_wstop bit for bit (verdict,
    iteration count, history, x, both true residuals) — on every engine that runs the size
    (graph passes on CSR / SELL slots / row classes, the one-CTA and cluster solvers via
    engine auto, CGS2, sharded), with and without weights."""
    s, val, b, dp = system(name, N, scal)
    _, _, d2 = oracle.gs_scale(s["row_ptr"], s["val"], s["b"], 2)
    w = None if scal == 2 else (d2 if dp is None else d2 / dp)
    A = gsk.CSR(s["row_ptr"], s["col"], val)
    maxit = 12 * m
    o = oracle.gmres(s["row_ptr"], s["col"], val, b, m, tol, maxit, weights=w, wstop=True)
    assert o[2]["iterations"] % m == 0 or o[2]["status"] != 0
    for kw in (dict(fmt="csr", engine="graph"), dict(fmt="sell", engine="graph"),
               dict(fmt="sell", engine="graph", sell_index="classes"), dict(fmt="csr"), dict(fmt="sell")):
        P = gsk.Plan(A, weights=w, gmres_wstop=True, **kw)
        assert_same_solve(P.gmres(b, m=m, tol=tol, maxit=maxit), o)
        P.close()
    P = gsk.Plan(A, fmt="sell", engine="graph", orth="cgs2", weights=w, gmres_wstop=True)
    assert_same_solve(P.gmres(b, m=m, tol=tol, maxit=maxit),
                      oracle.gmres(s["row_ptr"], s["col"], val, b, m, tol, maxit, weights=w, orth="cgs2", wstop=True))
    if s["n"] >= 4096:
        SP = gsk.ShardedPlan(A, shards=2, fmt="sell", weights=w, gmres_wstop=True)
        assert_same_solve(SP.gmres(b, m=m, tol=tol, maxit=maxit), o)
    # the default (estimate-stopped) runs are untouched by the option's existence
    P = gsk.Plan(A, fmt="sell", engine="graph", weights=w)
    assert_same_solve(P.gmres(b, m=m, tol=tol, maxit=maxit),
                      oracle.gmres(s["row_ptr"], s["col"], val, b, m, tol, maxit, weights=w))


def test_sharded_nccl_single_rank():
    """The multi-process code path (halo send/recv groups, ncclAllGather of the shard
    values, all inside the captured graphs) on a 1-rank NCCL communicator: bit-exact."""
    import ctypes
    lib = gsk.load()
    buf = ctypes.create_string_buffer(128)
    assert lib.gsk_nccl_unique_id(buf) == 0
    h = ctypes.c_void_p()
    assert lib.gsk_nccl_comm_create(ctypes.c_char_p(bytes(buf.raw)), 1, 0, ctypes.byref(h)) == 0

    class Comm:
        world, rank = 1, 0

    Comm.h = h
    s, val, b, _ = system("C3", 20, 2)
    A = gsk.CSR(s["row_ptr"], s["col"], val)
    for fmt in ("csr", "sell"):
        SP = gsk.ShardedPlan(A, fmt=fmt, comm=Comm)
        assert_same_solve(SP.bicgstab(b, tol=1e-9, maxit=400),
                          oracle.bicgstab(s["row_ptr"], s["col"], val, b, 1e-9, 400))
        assert_same_solve(SP.gmres(b, m=20, tol=1e-9, maxit=100),
                          oracle.gmres(s["row_ptr"], s["col"], val, b, 20, 1e-9, 100))
        SP.close()
    assert lib.gsk_nccl_comm_destroy(h) == 0


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("fmt", ["csr", "sell"])
def test_sharded_peer_reduce(P, fmt):
    """gsk_shard_opts.peer_reduce on one GPU (all shards in this process): every shard's
    finish stores its values into the gather buffer and releases its epoch flag, the
    global finish acquires the flags (already set: same stream) and reduces — the
    protocol of the multi-process path without the IPC mappings.  Bit-exact, over many
    epochs (both parities) and several solves on one plan."""
    s, val, b, _ = system("C3", 32, 2)  # 32768 rows: 8 shards of 4096, halos of one plane
    A = gsk.CSR(s["row_ptr"], s["col"], val)
    SP = gsk.ShardedPlan(A, shards=P, fmt=fmt, peer_reduce=True)
    ob = oracle.bicgstab(s["row_ptr"], s["col"], val, b, 1e-9, 400)
    og = oracle.gmres(s["row_ptr"], s["col"], val, b, 30, 1e-9, 100)
    for _ in range(2):
        assert_same_solve(SP.bicgstab(b, tol=1e-9, maxit=400), ob)
        assert_same_solve(SP.gmres(b, m=30, tol=1e-9, maxit=100), og)
    SP.close()


def test_sharded_local_input_single_rank():
    """gsk_shard_opts.local_input (each rank passes only its own rows, global columns;
    DESIGN.md §8 weak scaling) on a 1-rank NCCL communicator: the rows come from
    workloads.generate_rows, and the solve is bit-identical to the oracle on the whole
    system — here the stacked-slab workload C4w at reduced size."""
    import ctypes
    lib = gsk.load()
    buf = ctypes.create_string_buffer(128)
    assert lib.gsk_nccl_unique_id(buf) == 0
    h = ctypes.c_void_p()
    assert lib.gsk_nccl_comm_create(ctypes.c_char_p(bytes(buf.raw)), 1, 0, ctypes.byref(h)) == 0

    class Comm:
        world, rank = 1, 0

    Comm.h = h
    s = workloads.generate("C4w", N=16, param=2)
    loc = workloads.generate_rows("C4w", 0, s["n"], N=16, param=2)
    vo, bo, _ = oracle.gs_scale(s["row_ptr"], s["val"], s["b"], 2)
    A = gsk.CSR(loc["row_ptr"], loc["col"], loc["val"])
    As, bs, _ = gsk.gs_scale(A, loc["b"], 2)
    for fmt, peer in (("csr", False), ("sell", False), ("sell", True)):
        SP = gsk.ShardedPlan(As, fmt=fmt, comm=Comm, n_global=s["n"], peer_reduce=peer)
        assert_same_solve(SP.bicgstab(bs, tol=1e-9, maxit=300),
                          oracle.bicgstab(s["row_ptr"], s["col"], vo, bo, 1e-9, 300))
        assert_same_solve(SP.gmres(bs, m=30, tol=1e-9, maxit=90),
                          oracle.gmres(s["row_ptr"], s["col"], vo, bo, 30, 1e-9, 90))
        SP.close()
    assert lib.gsk_nccl_comm_destroy(h) == 0


def test_pass_order_does_not_change_results(tmp_path):
    """Alternating CTA order of consecutive passes (pass order and L2) keeps
    every partial in its slot: solves with GSK_ALT=0 (read once per process, hence the
    subprocess) are bit-identical to the default alternating order."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys, numpy as np; sys.path.insert(0, %r)\n"
        "import workloads, oracle, paper_0812_2769_b200 as gsk\n"
        "s = workloads.generate('C3', N=32); vo, bo, _ = oracle.gs_scale(s['row_ptr'], s['val'], s['b'], 2)\n"
        "P = gsk.Plan(gsk.CSR(s['row_ptr'], s['col'], vo), fmt='sell', engine='graph')\n"
        "x1, h1, _ = P.bicgstab(bo, tol=1e-8, maxit=300)\n"
        "x2, h2, _ = P.gmres(bo, m=30, tol=1e-8, maxit=120)\n"
        "np.savez(%r, x1=x1.cpu().numpy(), h1=h1, x2=x2.cpu().numpy(), h2=h2)\n"
    ) % (root, str(tmp_path / "alt.npz"))
    for alt in ("0", "1"):
        env = dict(os.environ, GSK_ALT=alt)
        subprocess.run([sys.executable, "-c", code.replace("alt.npz", "alt%s.npz" % alt)], check=True,
                       timeout=600, env=env)
    a = np.load(tmp_path / "alt0.npz")
    b = np.load(tmp_path / "alt1.npz")
    for k in ("x1", "h1", "x2", "h2"):
        assert np.array_equal(a[k], b[k]), k
    s = workloads.generate("C3", N=32)
    _, vo, bo, _ = system("C3", 32, 2)
    o = oracle.bicgstab(s["row_ptr"], s["col"], vo, bo, 1e-8, 300)
    assert np.array_equal(a["x1"], o[0])


def test_max_grid_512():
    """Maximum-size case: C4's recipe at 512³ (134 M rows, 938 M nonzeros; int32 indices
    hold up to 674³).  GS(2) and the first 3 Bi-CGSTAB iterations (SELL plan, the bench
    launch configuration) bit-exact against the oracle.  tools/max_grid.py runs the same
    up to 640³ (1.83 G nonzeros, 137 GB; profiles/r01_max_grid.jsonl)."""
    free, total = torch.cuda.mem_get_info()
    if total < 120 * 2**30:
        pytest.skip("needs a 180 GB B200")
    s = workloads.generate("C4", N=512)
    A = gsk.CSR.from_system(s)
    As, bs, _ = gsk.gs_scale(A, s["b"], 2)
    vo, bo, _ = oracle.gs_scale(s["row_ptr"], s["val"], s["b"], 2)
    assert np.array_equal(cpu(As.val), vo) and np.array_equal(cpu(bs), bo)
    del A
    P = gsk.Plan(As, fmt="sell")
    g = P.bicgstab(bs, tol=1e-8, maxit=3)
    o = oracle.bicgstab(s["row_ptr"], s["col"], vo, bo, 1e-8, 3)
    assert_same_solve(g, o)
