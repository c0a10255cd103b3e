"""Oracle pins (oracle/): each function checked against what the paper and the
mathematics fix, never against a retyped copy of itself.

  dot / wnorm2   exactness on integer data, the pairwise-tree shape on a hand-derived
                 case, the ceil(log2 n) u sum|q| error bound, thread-count invariance
  spmv           dense matvec; exact integer products
  gs_scale       Eq. (2) worked examples, unit L_p rows, solution invariance,
                 idempotence, errors
  sell_build     lossless round trip to CSR, window sort order, padding
  bicgstab/gmres dense LU on small systems, finite termination, Krylov least-squares
                 optimality, within-cycle monotonicity, A = I
"""
import json
import math
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import workloads

GOLD = os.path.join(os.path.dirname(__file__), "golden")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def csr_from_dense(A):
    n = A.shape[0]
    rp, col, val = [0], [], []
    for i in range(n):
        nz = np.nonzero(A[i])[0]
        col += list(nz)
        val += list(A[i, nz])
        rp.append(len(col))
    return np.array(rp, np.int32), np.array(col, np.int32), np.array(val, np.float64)


def dense(rp, col, val, n):
    A = np.zeros((n, n))
    for i in range(n):
        for k in range(rp[i], rp[i + 1]):
            A[i, col[k]] += val[k]
    return A


# ---------------------------------------------------------------- dot (AC-5)
def test_dot_exact_on_integers():
    rng = np.random.default_rng(1)
    for n in [1, 2, 3, 7, 1000, 4097, 100003]:
        a = rng.integers(-2 ** 20, 2 ** 20, n).astype(np.float64)
        b = rng.integers(-2 ** 12, 2 ** 12, n).astype(np.float64)
        exact = sum(int(x) * int(y) for x, y in zip(a, b))  # |sum| < 2^53
        assert oracle.dot(a, b) == float(exact)


def test_dot_tree_shape_hand_case():
    # (1e16 + 1) + (-1e16 + 1) rounds each pair to +-1e16 (ties-to-even), so the
    # pairwise tree gives 0 whereas left-to-right summation gives 1.
    a = np.array([1e16, 1.0, -1e16, 1.0])
    assert oracle.dot(a, np.ones(4)) == 0.0
    # 8 elements: ((x0+x1)+(x2+x3)) + ((x4+x5)+(x6+x7)); the right half cancels to 0,
    # the left half is 2^53 + 2 computed as (2^53 + 0) + (1 + 1) = 2^53 + 2.
    x = np.array([2.0 ** 53, 0.0, 1.0, 1.0, 1e300, -1e300, 5.0, -5.0])
    assert oracle.dot(x, np.ones(8)) == 2.0 ** 53 + 2
    # zero padding: n = 3 behaves as (x0 + x1) + (x2 + 0)
    y = np.array([2.0 ** 53, 1.0, 1.0])
    assert oracle.dot(y, np.ones(3)) == 2.0 ** 53  # (2^53+1 -> 2^53) + 1 -> 2^53


def test_dot_error_bound_and_signed_zero():
    rng = np.random.default_rng(2)
    n = 1 << 18
    a = rng.standard_normal(n) * np.exp(rng.uniform(-12, 12, n))
    b = rng.standard_normal(n)
    q = a * b
    ref = math.fsum(q)
    err = abs(oracle.dot(a, b) - ref)
    assert err <= math.ceil(math.log2(n)) * 2 ** -53 * np.abs(q).sum()
    assert math.copysign(1.0, oracle.dot(np.array([-0.0]), np.array([1.0]))) == 1.0  # T + 0.0


def test_wnorm2():
    r = np.array([3.0, 4.0, 12.0])
    assert oracle.wnorm2(r) == 169.0
    assert oracle.wnorm2(r, np.array([2.0, 0.5, 0.25])) == 36.0 + 4.0 + 9.0


def test_dot_thread_count_invariance():
    code = ("import sys; sys.path.insert(0, %r); import numpy as np, oracle, workloads;"
            "a = workloads.uniform(300001, 3, 9); b = workloads.uniform(300001, 4, 9);"
            "print(repr(oracle.dot(a, b)), oracle.num_threads())" % ROOT)
    outs = set()
    for t in ("1", "3", "8"):
        env = dict(os.environ, OMP_NUM_THREADS=t)
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                             text=True, check=True).stdout.split()
        assert out[1] == t
        outs.add(out[0])
    assert len(outs) == 1


# ---------------------------------------------------------------- spmv
def test_spmv_vs_dense():
    rng = np.random.default_rng(3)
    for n in [1, 5, 60, 200]:
        A = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.1)
        np.fill_diagonal(A, 1.0 + rng.random(n))
        rp, col, val = csr_from_dense(A)
        x = rng.standard_normal(n)
        y = oracle.spmv(rp, col, val, x)
        assert np.allclose(y, A @ x, rtol=1e-13, atol=1e-13 * np.abs(A).sum(1).max() * np.abs(x).max())


def test_spmv_exact_integers():
    s = workloads.generate("C3", N=10)
    rng = np.random.default_rng(4)
    val = rng.integers(-1000, 1000, s["nnz"]).astype(np.float64)
    x = rng.integers(-1000, 1000, s["n"]).astype(np.float64)
    y = oracle.spmv(s["row_ptr"], s["col"], val, x)
    A = dense(s["row_ptr"], s["col"], val, s["n"]).astype(np.int64)
    assert np.array_equal(y, (A @ x.astype(np.int64)).astype(np.float64))


# ---------------------------------------------------------------- GS(p), Eq. (2)
def ulps(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.abs(a.view(np.int64) - b.view(np.int64)).max() if a.size else 0


def test_gs_worked_examples():
    ex = json.load(open(os.path.join(GOLD, "gs_examples.json")))["examples"]
    for e in ex:
        n = len(e["rows"])
        A = np.zeros((n, max(max(c) for c in e["cols"]) + 1))
        for i in range(n):
            A[i, e["cols"][i]] = e["vals"][i]
        rp = np.array([0] + list(np.cumsum([len(c) for c in e["cols"]])), np.int32)
        val = np.concatenate([np.array(v, np.float64) for v in e["vals"]])
        vo, bo, d = oracle.gs_scale(rp, val, np.array(e["b"]), e["p"])
        if "scaled_vals" in e:
            assert ulps(vo, np.concatenate(e["scaled_vals"])) <= 1
            assert ulps(bo, e["scaled_b"]) <= 1
            assert ulps(d, e["d"]) <= 1
        if "norm" in e:
            assert ulps(1.0 / d, e["norm"]) <= 2


@pytest.mark.parametrize("name,N", [("C1", 32), ("C2", 64), ("C3", 16), ("C4", 16), ("C5", 64),
                                    ("P1", 40), ("P4", 12)])
@pytest.mark.parametrize("p", [1, 2, 3])
def test_gs_unit_row_norms(name, N, p):
    """After GS(p) every row has unit L_p norm: BASELINE north star
    asks 1e-14 relative."""
    s = workloads.generate(name, N=N)
    vo, bo, d = oracle.gs_scale(s["row_ptr"], s["val"], s["b"], p)
    rp = s["row_ptr"]
    a = np.abs(vo)
    sums = np.add.reduceat(a ** p, rp[:-1])
    norms = sums ** (1.0 / p)
    assert np.max(np.abs(norms - 1.0)) <= 1e-14
    # pattern preserved, b scaled by the same d
    assert np.all((vo == 0) == (s["val"] == 0))
    assert np.allclose(bo, s["b"] * d, rtol=0, atol=0)


def test_gs_solution_invariance_dense_lu():
    """GS leaves the solution of Ax=b unchanged (DAx = Db)."""
    for name, N in [("C1", 12), ("P1", 14), ("C4", 5), ("C2", 13)]:
        s = workloads.generate(name, N=N)
        A = dense(s["row_ptr"], s["col"], s["val"], s["n"])
        for p in (1, 2):
            vo, bo, _ = oracle.gs_scale(s["row_ptr"], s["val"], s["b"], p)
            DA = dense(s["row_ptr"], s["col"], vo, s["n"])
            x1 = np.linalg.solve(A, s["b"])
            x2 = np.linalg.solve(DA, bo)
            assert np.linalg.norm(x1 - x2) <= 1e-10 * np.linalg.norm(x1)


def test_gs_identity_idempotence_errors():
    n = 9
    rp = np.arange(n + 1, dtype=np.int32)
    vo, _, d = oracle.gs_scale(rp, np.ones(n), np.ones(n), 2)
    assert np.array_equal(vo, np.ones(n)) and np.array_equal(d, np.ones(n))
    s = workloads.generate("C2", N=32)
    v1, b1, _ = oracle.gs_scale(s["row_ptr"], s["val"], s["b"], 2)
    v2, b2, d2 = oracle.gs_scale(s["row_ptr"], v1, b1, 2)
    assert np.max(np.abs(v2 - v1) / np.abs(v1).clip(1e-300)) <= 4e-16 * 4
    assert np.max(np.abs(d2 - 1)) <= 4e-16 * 2
    with pytest.raises(ValueError):
        oracle.gs_scale(s["row_ptr"], s["val"], s["b"], 0)
    val = s["val"].copy()
    for r in (40, 17):
        val[s["row_ptr"][r]:s["row_ptr"][r + 1]] = 0.0
    with pytest.raises(oracle.ZeroRowError) as ei:
        oracle.gs_scale(s["row_ptr"], val, s["b"], 2)
    assert ei.value.row == 17  # smallest zero row


def test_gs1_bounds_spectrum():
    """GS(1): ||DA||_inf = 1, hence every eigenvalue has |lambda| <= 1."""
    s = workloads.generate("P1", N=20)
    vo, _, _ = oracle.gs_scale(s["row_ptr"], s["val"], s["b"], 1)
    DA = dense(s["row_ptr"], s["col"], vo, s["n"])
    assert np.abs(np.abs(DA).sum(1) - 1).max() < 1e-15
    assert np.abs(np.linalg.eigvals(DA)).max() <= 1 + 1e-12


# ---------------------------------------------------------------- SELL-C-sigma
@pytest.mark.parametrize("C,sigma", [(32, 256), (4, 8), (32, 32)])
def test_sell_round_trip(C, sigma):
    rng = np.random.default_rng(5)
    n = 1000
    lens = rng.integers(0, 9, n)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    col = np.concatenate([np.sort(rng.choice(n, l, replace=False)) for l in lens]).astype(np.int32)
    val = rng.standard_normal(rp[-1])
    S = oracle.sell_build(rp, col, val, C, sigma)
    S["roff"] = S["roff"].astype(np.int64)
    nch = (n + C - 1) // C
    assert S["chunk_ptr"][-1] == S["scol"].size
    seen = np.zeros(n, bool)
    for c in range(nch):
        L = S["chunk_len"][c]
        assert S["chunk_ptr"][c + 1] - S["chunk_ptr"][c] == L * C
        w0 = (c * C) // sigma * sigma
        lmax = 0
        for lane in range(C):
            row = w0 + S["roff"][c * C + lane]
            if row >= n:
                continue
            assert not seen[row]
            seen[row] = True
            ln = rp[row + 1] - rp[row]
            assert ln <= L
            lmax = max(lmax, ln)
            slots = S["chunk_ptr"][c] + np.arange(L) * C + lane
            assert np.array_equal(S["scol"][slots[:ln]], col[rp[row]:rp[row + 1]])
            assert np.array_equal(S["sval"][slots[:ln]], val[rp[row]:rp[row + 1]])
            assert np.all(S["scol"][slots[ln:]] == -1) and np.all(S["sval"][slots[ln:]] == 0)
        assert lmax == L  # chunk_len = the chunk's longest row
    assert seen.all()
    # within a window the sorted order is by descending length, ties by row id
    _check_window_order(S, rp, n, C, sigma)


def _chunk_slots(lens, C):
    return sum(max(lens[s:s + C]) for s in range(0, len(lens), C))


def _check_window_order(S, rp, n, C, sigma):
    """Per window: the rows in natural order when that needs no more padded slots than
    sorting them by descending length (ties by row id), else sorted (reading L1); either
    way the window's slot count is the sorted (minimal) one."""
    nch = (n + C - 1) // C
    roff = np.asarray(S["roff"], np.int64)
    naturals = 0
    for w0 in range(0, n, sigma):
        rows = [w0 + int(roff[s]) for s in range(w0, min(w0 + sigma, nch * C)) if w0 + roff[s] < n]
        lens = [int(rp[r + 1] - rp[r]) for r in range(w0, min(n, w0 + sigma))]
        srt = sorted(lens, reverse=True)
        if _chunk_slots(lens, C) <= _chunk_slots(srt, C):
            assert rows == list(range(w0, min(n, w0 + sigma)))
            naturals += 1
        else:
            key = [(-(rp[r + 1] - rp[r]), r) for r in rows]
            assert key == sorted(key)
        c0, c1 = w0 // C, (min(n, w0 + sigma) + C - 1) // C
        assert sum(S["chunk_len"][c0:c1]) == _chunk_slots(srt, C)
    return naturals


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "P4"])
def test_sell_stencil_windows_natural(name):
    """On the stencil systems sorting a window cannot save slots (its short boundary rows
    share a chunk with full rows either way), so every window keeps its natural order —
    and a window with a chunk of short rows is still sorted (constructed case)."""
    s = workloads.generate(name)
    S = oracle.sell_build(s["row_ptr"], s["col"], s["val"])
    nwin = (s["n"] + 255) // 256
    assert _check_window_order(S, s["row_ptr"], s["n"], 32, 256) == nwin
    lens = np.full(512, 7)
    lens[:32] = 3  # window 0: natural 3 + 7*7 = 52 slots / 32, sorted 7*7 + 3 = 52: natural
    lens[40] = 1
    lens[256:256 + 16] = 2
    lens[256 + 40:256 + 56] = 2  # window 1: natural 8*7 = 56, sorted 7*7 + 2 = 51: sorted
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    col = np.concatenate([np.arange(l) for l in lens]).astype(np.int32)
    S = oracle.sell_build(rp, col, np.ones(rp[-1]))
    assert _check_window_order(S, rp, 512, 32, 256) == 1
    assert list(S["roff"][256:256 + 32]) != list(range(32))


# ---------------------------------------------------------------- solvers
def small_system(n, seed, kappa=1e3):
    """Nonsymmetric D + S with diag D in [1, kappa] and ||S||_2 ~ 0.6, so the field of
    values lies in the right half plane and cond(A) <= ~kappa."""
    rng = np.random.default_rng(seed)
    d = np.geomspace(1.0, kappa, n)
    S = rng.standard_normal((n, n)) * (0.3 / np.sqrt(n))
    return np.diag(d) + S, rng.standard_normal(n)


@pytest.mark.parametrize("kappa", [30.0, 1e3])
@pytest.mark.parametrize("seed", range(6))
def test_solvers_match_dense_lu(seed, kappa):
    """n <= 200 with kappa in {30, 1e3}: GMRES (MGS, m = n and m = 15; CGS2 m = 15) and
    Bi-CGSTAB all match dense LU to 1e-10 relative (north star)."""
    n = [20, 50, 80, 120, 160, 200][seed]
    A, b = small_system(n, seed, kappa=kappa)
    assert np.linalg.cond(A) <= 1.1 * kappa
    rp, col, val = csr_from_dense(A)
    xs = np.linalg.solve(A, b)
    runs = [oracle.gmres(rp, col, val, b, n, 1e-14, 5 * n),
            oracle.gmres(rp, col, val, b, 15, 1e-14, 40 * n),
            oracle.gmres(rp, col, val, b, 15, 1e-14, 40 * n, orth="cgs2"),
            oracle.bicgstab(rp, col, val, b, 1e-14, 20 * n)]
    for x, h, rep in runs:
        assert rep["status"] == 0
        assert np.linalg.norm(x - xs) <= 1e-10 * np.linalg.norm(xs)


def test_identity_one_iteration():
    n = 50
    rp = np.arange(n + 1, dtype=np.int32)
    col = np.arange(n, dtype=np.int32)
    b = np.linspace(-1, 2, n)
    x, h, rep = oracle.bicgstab(rp, col, np.ones(n), b, 1e-12, 10)
    assert rep["status"] == 0 and rep["iterations"] == 1 and np.array_equal(x, b)
    x, h, rep = oracle.gmres(rp, col, np.ones(n), b, 5, 1e-12, 10)
    assert rep["status"] == 0 and rep["iterations"] == 1 and np.allclose(x, b, rtol=1e-15)


def test_finite_termination_diagonal():
    """Diagonal A with k distinct eigenvalues: Krylov dimension k, so GMRES(m>=k)
    converges in <= k steps and Bi-CGSTAB in <= k iterations (exact arithmetic)."""
    n = 300
    eigs = np.array([1.0, 2.5, 4.0, 7.0, 9.0])
    d = eigs[np.arange(n) % 5]
    rp = np.arange(n + 1, dtype=np.int32)
    col = np.arange(n, dtype=np.int32)
    b = workloads.uniform(n, 1, 1)
    x, h, rep = oracle.gmres(rp, col, d, b, 10, 1e-12, 100)
    assert rep["status"] == 0 and rep["iterations"] <= 5
    x, h, rep = oracle.bicgstab(rp, col, d, b, 1e-12, 100)
    assert rep["status"] == 0 and rep["iterations"] <= 5
    assert np.allclose(x, b / d, rtol=1e-10)


@pytest.mark.parametrize("orth", ["mgs", "cgs2"])
def test_gmres_is_krylov_least_squares(orth):
    """hist[j] * ||r0|| = min over x in x0 + K_j(A, r0) of ||b - A x|| (GMRES's
    defining property, Saad & Schultz 1986); checked by brute-force least squares
    on an orthonormalised explicit Krylov basis.  Holds for either orthogonalisation
    (MGS, or AZTEC's double classical Gram-Schmidt)."""
    n = 60
    A, b = small_system(n, 11, kappa=10.0)
    rp, col, val = csr_from_dense(A)
    x, h, rep = oracle.gmres(rp, col, val, b, n, 1e-15, n, orth=orth)
    beta0 = np.linalg.norm(b)
    K = [b / beta0]
    for j in range(1, 30):  # K_j = span{r0, A r0, ..., A^{j-1} r0}
        Q, _ = np.linalg.qr(np.array(K).T)
        K.append(A @ Q[:, -1])
        y, *_ = np.linalg.lstsq(A @ Q, b, rcond=None)
        best = np.linalg.norm(b - A @ Q @ y)
        assert abs(h[j] * beta0 - best) <= 1e-8 * beta0 + 1e-6 * best, j


def test_gmres_nonincreasing_within_cycle():
    s = workloads.generate("C1")
    vo, bo, _ = oracle.gs_scale(s["row_ptr"], s["val"], s["b"], 2)
    m = 20
    x, h, rep = oracle.gmres(s["row_ptr"], s["col"], vo, bo, m, 1e-8, 400)
    assert rep["restarts"] >= 10
    for c0 in range(0, len(h) - 1, m):
        seg = h[c0 + 1:c0 + m + 1] if c0 else h[0:m + 1]
        assert np.all(np.diff(seg) <= np.spacing(seg[:-1]))  # 1-ulp slack (reading B13)


def test_true_relres_recomputed():
    """Frame consistency: the reported true residual is ||b - A x|| / ||b - A x0||."""
    s = workloads.generate("C2", N=48)
    vo, bo, _ = oracle.gs_scale(s["row_ptr"], s["val"], s["b"], 2)
    for solve in ("bicgstab", "gmres"):
        if solve == "bicgstab":
            x, h, rep = oracle.bicgstab(s["row_ptr"], s["col"], vo, bo, 1e-9, 3000)
        else:
            x, h, rep = oracle.gmres(s["row_ptr"], s["col"], vo, bo, 30, 1e-9, 3000)
        DA = dense(s["row_ptr"], s["col"], vo, s["n"])
        tr = np.linalg.norm(bo - DA @ x) / np.linalg.norm(bo)
        assert abs(tr - rep["true_relres"]) <= 1e-6 * tr + 1e-15
        assert rep["history_len"] == len(h) == rep["iterations"] + 1


def test_breakdown_on_exact_zero_sigma():
    """Bi-CGSTAB breakdown (exact-zero reading B5): a skew
    system with r0 orthogonal to A r0 gives sigma = <r0, A r0> = 0 at iteration 1."""
    A = np.array([[0.0, 1.0], [-1.0, 0.0]])
    rp, col, val = csr_from_dense(A)
    x, h, rep = oracle.bicgstab(rp, col, val, np.array([1.0, 0.0]), 1e-10, 10)
    assert rep["status"] == 2 and rep["breakdown_at"] == 1 and rep["iterations"] == 0


def test_zero_rhs_converges_immediately():
    s = workloads.generate("C1", N=8)
    b = np.zeros(s["n"])
    for f in (oracle.bicgstab, ):
        x, h, rep = f(s["row_ptr"], s["col"], s["val"], b, 1e-8, 10)
        assert rep["status"] == 0 and rep["iterations"] == 0 and np.all(x == 0)
    x, h, rep = oracle.gmres(s["row_ptr"], s["col"], s["val"], b, 5, 1e-8, 10)
    assert rep["status"] == 0 and rep["iterations"] == 0


# ---------------------------------------------------------------- two-sided scaling
def test_two_sided_scaling():
    """D^1/2 A D^1/2 y = D^1/2 b, x = D^1/2 y: the solution is
    unchanged, symmetry of A is kept (to 1 ulp: the two factors round in a fixed
    order), and for p = 2 the entries are a_ij / sqrt(||a_i|| ||a_j||)."""
    for name, N in [("P1", 14), ("C3", 6), ("lap2d", 9)]:
        s = workloads.generate(name, N=N)
        A = dense(s["row_ptr"], s["col"], s["val"], s["n"])
        v2, b2, sv = oracle.gs_scale_sym(s["row_ptr"], s["col"], s["val"], s["b"], 2)
        A2 = dense(s["row_ptr"], s["col"], v2, s["n"])
        nrm = np.sqrt((A ** 2).sum(1))
        assert np.allclose(sv, 1 / np.sqrt(nrm), rtol=1e-15, atol=0)
        assert np.allclose(A2, A / np.sqrt(np.outer(nrm, nrm)), rtol=2e-15, atol=0)
        y = np.linalg.solve(A2, b2)
        x = oracle.unscale(sv, y)
        xs = np.linalg.solve(A, s["b"])
        assert np.linalg.norm(x - xs) <= 1e-10 * np.linalg.norm(xs)
        if name == "lap2d":
            assert np.abs(A2 - A2.T).max() <= 2.3e-16 * np.abs(A2).max()
    with pytest.raises(ValueError):
        oracle.gs_scale_sym(s["row_ptr"], s["col"], s["val"], s["b"], 0)


def test_sell_dict_round_trip():
    """SELL-D (the GPU's column-index dictionary): decoding row + dict_c[idx] gives back
    every column of the SELL layout; padding stays marked; dictionaries are ascending
    and unique; the permuted C5 system (random deltas) is rejected."""
    for name, N in [("C4", 16), ("C3", 12), ("C2", 40), ("C1", None)]:
        s = workloads.generate(name, N=N)
        S = oracle.sell_build(s["row_ptr"], s["col"], s["val"])
        D = oracle.sell_dict(s["n"], S)
        assert D is not None
        nch = S["chunk_len"].size
        for c in range(nch):
            dct = D["dict"][D["dict_ptr"][c]:D["dict_ptr"][c + 1]]
            assert np.all(np.diff(dct) > 0) and dct.size <= 32
            w0 = (c * 32) // 256 * 256
            for k in range(S["chunk_len"][c]):
                for lane in range(32):
                    slot = S["chunk_ptr"][c] + 32 * k + lane
                    idx = int(D["sidx"][slot])
                    if S["scol"][slot] < 0:
                        assert idx == 255
                    else:
                        assert w0 + int(S["roff"][c * 32 + lane]) + dct[idx] == S["scol"][slot]
    s = workloads.generate("C5", N=64)
    assert oracle.sell_dict(s["n"], oracle.sell_build(s["row_ptr"], s["col"], s["val"])) is None


# ---------------------------------------------------------------- verdict branches
VERDICTS = json.load(open(os.path.join(GOLD, "verdict_systems.json")))["cases"]


def _val(s):
    from fractions import Fraction
    if s == "nan":
        return float("nan")
    if s.startswith("sqrt:"):
        return math.sqrt(Fraction(s[5:]))
    return float(Fraction(s))


@pytest.mark.parametrize("case", VERDICTS, ids=[c["name"] for c in VERDICTS])
def test_verdict_branches_hand_derived(case):
    """Every termination branch of both solvers (readings B4/B5/B8)
    on a tiny system whose iterates were derived by hand in exact arithmetic
    (tests/golden/verdict_systems.json gives each derivation): one full Bi-CGSTAB
    iteration (alpha = 5/22, omega = 13/50, x1 = (73, 276)/550), one GMRES step,
    the ||s|| half-step exit, exact rho = 0 / sigma = 0 / <t,t> = 0 / omega = 0
    breakdowns and the non-finite DIVERGED exit."""
    A = np.array(case["A"], np.float64)
    b = np.array(case["b"], np.float64)
    rp, col, val = csr_from_dense(A)
    if case["solver"] == "bicgstab":
        x, h, rep = oracle.bicgstab(rp, col, val, b, case["tol"], case["maxit"])
    else:
        x, h, rep = oracle.gmres(rp, col, val, b, case["m"], case["tol"], case["maxit"])
    e = case["expect"]
    assert (rep["status"], rep["iterations"], rep["breakdown_at"]) == (e["status"], e["iterations"],
                                                                        e["breakdown_at"])
    want = np.array([_val(v) for v in e["hist"]])
    assert h.shape == want.shape
    assert np.allclose(h, want, rtol=1e-14, atol=0, equal_nan=True), (h, want)
    if "x" in e:
        xw = np.array([_val(v) for v in e["x"]])
        assert np.allclose(x, xw, rtol=1e-14, atol=1e-300), (x, xw)
    if e["status"] == 3:
        assert not np.isfinite(rep["relres"])


# ---------------------------------------------------------------- SELL-U
def _decode_uniform(U, S, rp, n, C=32, sigma=256, maxu=8):
    """Rows rebuilt from a SELL-U encoding: {row: [(col, val), ...]} in slot order."""
    rows = {}
    nch = (n + C - 1) // C
    roff = np.asarray(S["roff"], np.int64)
    for c in range(nch):
        w0 = (c * C) // sigma * sigma
        L = (U["uptr"][c + 1] - U["uptr"][c]) // C
        for lane in range(C):
            row = w0 + int(roff[c * C + lane])
            if row >= n:
                continue
            ent = []
            for k in range(L):
                v = U["uval"][U["uptr"][c] + k * C + lane]
                if (int(U["umask"][c * maxu + k]) >> lane) & 1:
                    ent.append((row + int(U["udel"][c * maxu + k]), v))
                else:
                    assert v == 0.0
            rows[row] = ent
    return rows


@pytest.mark.parametrize("name,N", [("C1", None), ("C2", 64), ("C3", 16), ("C4", 20), ("P4", 12), ("lap3d", 16)])
def test_sell_uniform_round_trip(name, N):
    """SELL-U (chunk-uniform column deltas): decoding every masked slot gives
    back each row's CSR entries in ascending column order (so the SpMV chain is AC-3's),
    deltas ascend, unused entries are zero, and on the stencil systems a chunk has exactly
    as many deltas as its longest row — the same slot count as SELL-C-sigma."""
    s = workloads.generate(name, N=N)
    S = oracle.sell_build(s["row_ptr"], s["col"], s["val"])
    U = oracle.sell_uniform(s["row_ptr"], s["col"], s["val"], S)
    assert U is not None
    rows = _decode_uniform(U, S, s["row_ptr"], s["n"])
    rp = s["row_ptr"]
    for r in range(s["n"]):
        ent = rows[r]
        assert [c for c, _ in ent] == list(s["col"][rp[r]:rp[r + 1]])
        assert np.array_equal([v for _, v in ent], s["val"][rp[r]:rp[r + 1]])
    nch = (s["n"] + 31) // 32
    for c in range(nch):
        L = (U["uptr"][c + 1] - U["uptr"][c]) // 32
        d = U["udel"][c * 8:c * 8 + L]
        assert np.all(np.diff(d) > 0) and np.all(U["udel"][c * 8 + L:c * 8 + 8] == 0)
        assert np.all(U["umask"][c * 8 + L:c * 8 + 8] == 0) and np.all(U["umask"][c * 8:c * 8 + L] != 0)
    # a chunk holds at least its longest row's slots; where a window keeps its natural
    # order (every window of the full-size stencil configs) exactly that many, so the
    # layout has SELL-C-sigma's slot count; sorted boundary windows of these small grids
    # mix rows missing different neighbours (a few % more slots)
    L = np.diff(U["uptr"]) // 32
    assert np.all(L >= S["chunk_len"])
    nat = _check_window_order(S, rp, s["n"], 32, 256) == (s["n"] + 255) // 256
    assert (U["uptr"][-1] == S["chunk_ptr"][-1]) if nat else (U["uptr"][-1] <= 1.05 * S["chunk_ptr"][-1])


def test_sell_uniform_inapplicable_and_constructed():
    """A chunk with more than 8 distinct deltas (the permuted C5 system) makes SELL-U
    inapplicable; a hand-built 2-chunk system pins the encoding exactly."""
    s = workloads.generate("C5", N=64)
    S = oracle.sell_build(s["row_ptr"], s["col"], s["val"])
    assert oracle.sell_uniform(s["row_ptr"], s["col"], s["val"], S) is None
    # 40 rows: row r has entries at r-1 (r>0), r, r+3 (r+3<40); values 10r + k
    cols, vals, rp = [], [], [0]
    for r in range(40):
        cc = [c for c in (r - 1, r, r + 3) if 0 <= c < 40]
        cols += cc
        vals += [10.0 * r + k for k in range(len(cc))]
        rp.append(len(cols))
    S = oracle.sell_build(np.array(rp), np.array(cols), np.array(vals))
    U = oracle.sell_uniform(np.array(rp), np.array(cols), np.array(vals), S)
    assert list(U["uptr"]) == [0, 96, 192] and list(U["udel"][:3]) == [-1, 0, 3] and list(U["udel"][8:11]) == [-1, 0, 3]
    assert U["umask"][0] == 0xFFFFFFFE and U["umask"][1] == 0xFFFFFFFF and U["umask"][2] == 0xFFFFFFFF
    assert U["umask"][8] == 0xFF and U["umask"][9] == 0xFF and U["umask"][10] == 0x1F  # rows 32..39; r+3 < 40 for r <= 36
    assert U["uval"][0] == 0.0 and U["uval"][32] == 0.0 and U["uval"][64] == 1.0  # row 0: (0 -> 0.0), (3 -> 1.0)
    assert U["uval"][1] == 10.0 and U["uval"][33] == 11.0 and U["uval"][65] == 12.0


@pytest.mark.parametrize("kind,k", [("rho0", 10), ("omega0", 10), ("nan", 10), ("rho0", 1), ("nan", 90)])
def test_fault_hook_verdicts(kind, k):
    """Test-only fault hook (the GPU mirrors it with GSK_FAULT): forcing rho = 0
    at the end of iteration k gives BREAKDOWN at k + 1, omega = 0 in iteration k gives
    BREAKDOWN at k (after the x, r update, reading B5), NaN in r_0 gives DIVERGED at k; the
    history before the fault is the un-faulted run's, and clearing the hook restores it."""
    s = workloads.generate("C1")
    vo, bo, _ = oracle.gs_scale(s["row_ptr"], s["val"], s["b"], 2)
    x0, h0, r0 = oracle.bicgstab(s["row_ptr"], s["col"], vo, bo, 1e-8, 2000)
    try:
        oracle.set_fault(kind, k)
        x, h, rep = oracle.bicgstab(s["row_ptr"], s["col"], vo, bo, 1e-8, 2000)
    finally:
        oracle.set_fault()
    want = {"rho0": (2, k, k + 1), "omega0": (2, k, k), "nan": (3, k, 0)}[kind]
    assert (rep["status"], rep["iterations"], rep["breakdown_at"]) == want
    assert np.array_equal(h[:k], h0[:k])
    if kind == "rho0":
        assert np.array_equal(h, h0[:k + 1])
    if kind == "nan":
        assert np.isnan(h[k])
    x2, h2, _ = oracle.bicgstab(s["row_ptr"], s["col"], vo, bo, 1e-8, 2000)
    assert np.array_equal(h2, h0) and np.array_equal(x2, x0)


def _decode_classes(R, n):
    """CSR arrays decoded from a row-class dictionary."""
    rp, cols, vals = [0], [], []
    for r in range(n):
        k = int(R["cls"][r])
        L = int(R["len"][k])
        cols += [r + int(d) for d in R["delta"][k, :L]]
        vals += list(R["val"][k, :L])
        rp.append(len(cols))
    return np.array(rp), np.array(cols), np.array(vals)


@pytest.mark.parametrize("name,N,p,ncls", [("C1", None, 2, 14), ("C3", 16, 2, None), ("C4", 20, 0, None),
                                           ("C4", 64, 2, 99), ("P4", 12, 1, None), ("lap3d", 8, 0, 27)])
def test_row_classes_round_trip(name, N, p, ncls):
    """Row-class dictionary (oracle.cpp "RCD"; the paper's piecewise-constant problems,
    PAPER.md:269-294): lossless — decoding cls + dictionary gives back every row's columns
    and bit-identical values in CSR order; classes are numbered by first occurrence; the
    class count is what the geometry fixes (a Laplacian on a box: 3^3 boundary types; C1:
    pinned by an independent np.unique over (len, deltas, value bits))."""
    s = workloads.generate(name, N=N)
    val = oracle.gs_scale(s["row_ptr"], s["val"], s["b"], p)[0] if p else s["val"]
    R = oracle.row_classes(s["row_ptr"], s["col"], val)
    assert R is not None
    rp, cols, vals = _decode_classes(R, s["n"])
    assert np.array_equal(rp, s["row_ptr"]) and np.array_equal(cols, s["col"])
    assert np.array_equal(vals.view(np.uint64), np.ascontiguousarray(val).view(np.uint64))
    # first-occurrence numbering: the first row of class k has no smaller class after it
    first = np.full(len(R["len"]), s["n"])
    np.minimum.at(first, R["cls"], np.arange(s["n"]))
    assert np.all(np.diff(first) > 0) and first[0] == 0
    # unused dictionary places are zero
    for k, L in enumerate(R["len"]):
        assert np.all(R["delta"][k, L:] == 0) and np.all(R["val"][k, L:] == 0.0)
    # independent count of the distinct rows
    ln = np.diff(s["row_ptr"])
    K = 8
    key = np.zeros((s["n"], 1 + 2 * K), np.uint64)
    rows = np.repeat(np.arange(s["n"]), ln)
    pos = np.arange(len(s["col"])) - np.repeat(s["row_ptr"][:-1], ln)
    key[:, 0] = ln
    key[rows, 1 + pos] = (s["col"] - rows).astype(np.int64).view(np.uint64)
    key[rows, 1 + K + pos] = np.ascontiguousarray(val).view(np.uint64)
    assert len(np.unique(key, axis=0)) == len(R["len"])
    if ncls is not None:
        assert len(R["len"]) == ncls


def test_row_classes_constructed_and_inapplicable():
    """A hand-built system pins the encoding entry by entry; -0.0 and +0.0 are different
    values (bit patterns, not ==); a row longer than maxlen, or more classes than maxcls
    (C2: the velocity depends on the node), make the format inapplicable."""
    # 6 rows: entries (r-1: -1.0), (r: d_r), (r+1: -1.0) inside [0, 6); d = 2,2,2,3,2,2
    d = [2.0, 2.0, 2.0, 3.0, 2.0, 2.0]
    rp, cols, vals = [0], [], []
    for r in range(6):
        for c, v in ((r - 1, -1.0), (r, d[r]), (r + 1, -1.0)):
            if 0 <= c < 6:
                cols.append(c)
                vals.append(v)
        rp.append(len(cols))
    R = oracle.row_classes(np.array(rp), np.array(cols), np.array(vals), maxlen=4)
    # classes by first occurrence: 0 = first row (no left), 1 = interior d=2, 2 = d=3, 3 = last row
    assert list(R["cls"]) == [0, 1, 1, 2, 1, 3]
    assert list(R["len"]) == [2, 3, 3, 2]
    assert R["delta"].tolist() == [[0, 1, 0, 0], [-1, 0, 1, 0], [-1, 0, 1, 0], [-1, 0, 0, 0]]
    assert R["val"].tolist() == [[2.0, -1.0, 0, 0], [-1.0, 2.0, -1.0, 0], [-1.0, 3.0, -1.0, 0], [-1.0, 2.0, 0, 0]]
    # signed zero: row 4's diagonal -0.0 vs row 1's would-be +0.0 are distinct classes
    v2 = np.array(vals)
    v2[rp[1] + 1] = 0.0
    v2[rp[2] + 1] = -0.0
    R2 = oracle.row_classes(np.array(rp), np.array(cols), v2, maxlen=4)
    assert R2["cls"][1] != R2["cls"][2]
    assert oracle.row_classes(np.array(rp), np.array(cols), np.array(vals), maxlen=2) is None
    assert oracle.row_classes(np.array(rp), np.array(cols), np.array(vals), maxlen=4, maxcls=3) is None
    s = workloads.generate("C2", N=96)
    assert oracle.row_classes(s["row_ptr"], s["col"], s["val"]) is None


def test_gmres_weighted_stop_at_cycle_ends():
    """Reading B2w (the relative residual "always" measured on the
    GS(2)-scaled system): with wstop the least-squares estimate no longer stops GMRES; the
    run ends CONVERGED at the first cycle end whose weighted TRUE residual is below tol.
    Pinned independently of the oracle's own stopping code: cycle ends are found by running
    the plain solver with maxit = k m (iterates do not depend on tol or maxit, B11) and
    the weighted residual of each is recomputed with numpy."""
    s = workloads.generate("C1")
    rp, col, val, b = s["row_ptr"], s["col"], s["val"], s["b"]
    v1, b1, d1 = oracle.gs_scale(rp, val, b, 1)
    _, _, d2 = oracle.gs_scale(rp, val, b, 2)
    w = d2 / d1  # GS(2) frame of the GS(1)-scaled system
    m, tol = 20, 1e-4
    A = np.zeros((s["n"], s["n"]))
    for i in range(s["n"]):
        A[i, col[rp[i]:rp[i + 1]]] = v1[rp[i]:rp[i + 1]]
    n0w = np.linalg.norm(w * b1)
    first = None
    for k in range(1, 8):
        xk, hk, rk = oracle.gmres(rp, col, v1, b1, m, 1e-300, k * m)
        if np.linalg.norm(w * (b1 - A @ xk)) / n0w < tol:
            first = k
            break
    assert first is not None and first > 1
    x, h, r = oracle.gmres(rp, col, v1, b1, m, tol, 2000, weights=w, wstop=True)
    assert r["status"] == 0 and r["iterations"] == first * m and r["restarts"] == first - 1
    assert np.array_equal(x, xk) and np.array_equal(h, hk)  # the same iterates and estimates
    assert r["true_relres_w"] < tol
    assert abs(r["true_relres_w"] - np.linalg.norm(w * (b1 - A @ x)) / n0w) <= 1e-12 * r["true_relres_w"] + 1e-18
    # the estimate alone stops earlier, mid-cycle (B1), and its history is a prefix
    x0, h0, r0 = oracle.gmres(rp, col, v1, b1, m, tol, 2000, weights=w)
    assert r0["status"] == 0 and r0["iterations"] < r["iterations"] and r0["iterations"] % m != 0
    assert np.array_equal(h0, h[:len(h0)])
    # without weights wstop tests the plain true residual at cycle ends
    xu, hu, ru = oracle.gmres(rp, col, v1, b1, m, tol, 2000, wstop=True)
    assert ru["status"] == 0 and ru["iterations"] % m == 0 and ru["true_relres"] < tol


def test_gmres_weighted_stop_refuses_the_unscaled_estimate():
    """The advisor's case: unscaled C1, tol 1e-3.  The least-squares estimate (unscaled
    frame) crosses tol at step 19 while the GS(2)-frame residual is still 0.84; with wstop
    the run is not CONVERGED (MAXIT, GS(2)-frame residual >= tol)."""
    s = workloads.generate("C1")
    rp, col, val, b = s["row_ptr"], s["col"], s["val"], s["b"]
    _, _, d2 = oracle.gs_scale(rp, val, b, 2)
    _, _, r0 = oracle.gmres(rp, col, val, b, 20, 1e-3, 600, weights=d2)
    assert r0["status"] == 0 and r0["iterations"] == 19 and r0["true_relres_w"] > 0.5
    _, h, r = oracle.gmres(rp, col, val, b, 20, 1e-3, 600, weights=d2, wstop=True)
    assert r["status"] == 1 and r["iterations"] == 600 and r["true_relres_w"] >= 1e-3
    assert h.min() < 1e-3  # the estimate did cross
