"""Generator pins (workloads/, shared input module).

The generator discretises the paper's PDEs (§2.1) and
BASELINE.json's configs; these tests pin it to closed forms and to the
eigenvalue table tbl1b.
"""
import json
import os

import numpy as np
import pytest

import workloads

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def dense(s):
    n = s["n"]
    A = np.zeros((n, n))
    for i in range(n):
        for k in range(s["row_ptr"][i], s["row_ptr"][i + 1]):
            A[i, s["col"][k]] += s["val"][k]
    return A


@pytest.mark.parametrize("name,N,dim", [("C1", 32, 2), ("C2", 40, 2), ("C3", 12, 3), ("C4", 16, 3),
                                        ("C5", 48, 2), ("P1", 20, 2), ("P4", 10, 3),
                                        ("lap2d", 9, 2), ("lap3d", 7, 3)])
def test_csr_invariants_and_nnz_closed_form(name, N, dim):
    s = workloads.generate(name, N=N)
    n, nnz = s["n"], s["nnz"]
    assert n == N ** dim
    # 5N^2-4N (2D 5-point) and 7N^3-6N^2 (3D 7-point) with Dirichlet rows eliminated
    assert nnz == (5 * N * N - 4 * N if dim == 2 else 7 * N ** 3 - 6 * N * N)
    rp, col = s["row_ptr"], s["col"]
    assert rp[0] == 0 and rp[-1] == nnz and np.all(np.diff(rp) >= 1)
    assert np.all(np.diff(rp) <= 2 * dim + 1)        # stencil locality
    for i in range(n):
        c = col[rp[i]:rp[i + 1]]
        assert np.all(np.diff(c) > 0) and c.min() >= 0 and c.max() < n
        assert i in c                                   # structural diagonal
    assert np.all(np.isfinite(s["val"]))


def test_full_size_dims():
    # BASELINE.json configs: n and nnz at full size (SURVEY §8 size table)
    assert workloads.dims(1, 32) == (1024, 4992)
    assert workloads.dims(2, 512) == (262144, 1308672)
    assert workloads.dims(3, 128) == (2097152, 14581760)
    assert workloads.dims(4, 256) == (16777216, 117047296)
    assert workloads.dims(5, 2048) == (4194304, 20963328)


@pytest.mark.parametrize("name,N", [("lap2d", 15), ("lap3d", 9)])
def test_laplacian_closed_form_eigenvectors(name, N):
    """k=1, no convection: A phi = lambda phi with phi = prod sin(p_a pi x_a) and
    lambda = sum_a (2 - 2 cos(p_a pi h)) for the h^2-scaled operator (reading M2)."""
    s = workloads.generate(name, N=N)
    A = dense(s)
    assert np.allclose(A, A.T, rtol=0, atol=0)
    h = 1.0 / (N + 1)
    coords = (np.arange(N) + 1) * h
    dim = 2 if name == "lap2d" else 3
    for ps in [(1, 1, 1), (2, 3, 1), (N, 1, 2)]:
        grids = np.meshgrid(*[np.sin(ps[a] * np.pi * coords) for a in range(dim)], indexing="ij")
        phi = np.ones_like(grids[0])
        for g in grids:
            phi = phi * g
        phi = phi.transpose().reshape(-1)  # x fastest
        lam = sum(2 - 2 * np.cos(ps[a] * np.pi * h) for a in range(dim))
        assert np.allclose(A @ phi, lam * phi, rtol=0, atol=1e-12)
    # interior rows sum to 0, boundary rows positive (S:340-style check)
    rs = A.sum(axis=1)
    assert np.all(rs >= -1e-12) and np.isclose(rs.min(), 0.0) and rs.max() > 0


def test_c1_coefficients_by_hand():
    """C1 (BASELINE configs[0]): k=1e4 strictly inside (1/4,3/4)^2, b=(10,10), centred.
    Row of the interior node (I,J)=(16,16): all four faces inside -> diagonal 4e4,
    off-diagonals -1e4 -+ 10*h/2."""
    s = workloads.generate("C1")
    N, h = 32, 1.0 / 33
    r = 16 + N * 16
    cols = s["col"][s["row_ptr"][r]:s["row_ptr"][r + 1]]
    vals = s["val"][s["row_ptr"][r]:s["row_ptr"][r + 1]]
    assert list(cols) == [r - N, r - 1, r, r + 1, r + N]
    c = 10 * h * 0.5
    assert np.allclose(vals, [-1e4 - c, -1e4 - c, 4e4, -1e4 + c, -1e4 + c], rtol=1e-15)
    # corner node (0,0): k = 1 on all faces
    vals0 = s["val"][0:3]
    assert np.allclose(vals0, [4.0, -1 + c, -1 + c], rtol=1e-15)


def test_c4_slabs_and_upwind():
    s = workloads.generate("C4", N=32)
    A_diag = []
    N = 32
    for K in range(N):
        r = 5 + N * 5 + N * N * K
        ks = s["val"][s["row_ptr"][r]:s["row_ptr"][r + 1]]
        A_diag.append(ks)
    # x-y faces of a node take the slab of the node; k values drawn from the list
    allowed = {1.0, 1e2, 1e4, 1e-2, 1e6}
    # west off-diagonal = -k - b_x h (upwind, b_x = 30 > 0); east = -k (no convection)
    h = 1.0 / (N + 1)
    for ks in A_diag:
        k_east = -ks[4]
        assert k_east in allowed
    seen = {-ks[4] for ks in A_diag}
    assert len(seen) == 5  # all five slabs present, cuts in [1, N-1]


def test_c5_permutation_is_symmetric_relabel():
    s = workloads.generate("C5", N=24)
    u = workloads.generate("C5", N=24, param=-1.0)  # unpermuted
    pi = s["perm"]
    n = s["n"]
    assert np.array_equal(np.sort(pi), np.arange(n))
    Ap, Au = dense(s), dense(u)
    assert np.array_equal(Ap[np.ix_(pi, pi)], Au)
    assert np.array_equal(s["xstar"][pi], u["xstar"])
    # k log-uniform in [1e-3, 1e5]: h^2-scaled diagonal = sum of 4 face k
    assert np.all(np.diag(Au) > 4e-3 - 1e-9) and np.all(np.diag(Au) < 4e5 + 1)


def test_rhs_is_A_xstar():
    s = workloads.generate("C3", N=10)
    A = dense(s)
    assert np.allclose(A @ s["xstar"], s["b"], rtol=1e-13, atol=1e-9)
    assert s["xstar"].min() >= -1 and s["xstar"].max() < 1
    p1 = workloads.generate("P1", N=12)
    assert np.array_equal(p1["xstar"], np.ones(144))


def test_determinism():
    a = workloads.generate("C2", N=64)
    b = workloads.generate("C2", N=64)
    for k in ("row_ptr", "col", "val", "b", "xstar"):
        assert np.array_equal(a[k], b[k])
    c = workloads.generate("C2", N=64, seed=7)
    assert not np.array_equal(a["val"], c["val"]) or not np.array_equal(a["xstar"], c["xstar"])


def _eig_stats(A):
    lam = np.linalg.eigvals(A)
    mods = np.abs(lam)
    re = lam.real
    hist, _ = np.histogram(re, bins=100, range=(re.min(), re.max()))
    return mods.min(), mods.max(), hist[0], np.abs(lam.imag).max()


@pytest.mark.slow
def test_paper_tbl1b_eigenvalues():
    """Table tbl1b: P1 on a 40x40 grid.  Pins readings M1
    (h = 1/(N+1)), M2 (h^2 scaling), M3 (face-midpoint k) and, through GS(2), Eq. (2)."""
    import oracle
    gold = json.load(open(os.path.join(GOLD, "paper_tables.json")))["tbl1b"]
    s = workloads.generate("P1", N=40)
    lmin, lmax, first, _ = _eig_stats(dense(s))
    g = gold["original"]
    assert first == g["first_bin"]
    assert abs(lmax - g["lmax"]) / g["lmax"] < 0.005
    assert abs(lmin - g["lmin"]) / g["lmin"] < 0.02
    vo, _, _ = oracle.gs_scale(s["row_ptr"], s["val"], s["b"], 2)
    sg = dict(s, val=vo)
    lmin, lmax, first, _ = _eig_stats(dense(sg))
    g = gold["gs"]
    assert first == g["first_bin"]
    assert abs(lmax - g["lmax"]) / g["lmax"] < 0.005
    assert abs(lmin - g["lmin"]) / g["lmin"] < 0.005
    c = workloads.generate("P1cont", N=40)
    lmin, lmax, first, imag = _eig_stats(dense(c))
    g = gold["cont"]
    assert first == g["first_bin"]
    assert abs(lmax - g["lmax"]) / g["lmax"] < 0.005
    assert abs(lmin - g["lmin"]) / g["lmin"] < 0.005
    # "all real in (0, 8000)"; closed form 1000(4-2cos(pi h)-2cos(pi h))
    assert imag < 1e-6 * lmax


@pytest.mark.parametrize("N", [6, 10])
def test_stacked_slabs(N):
    """C4w (weak scaling): G = 1 is C4 exactly; G copies have the closed-form
    nnz 7 N^2 Nz - 4 N Nz - 2 N^2 (Nz = G N); row blocks from generate_rows (what each
    rank builds) concatenate to the whole system; a block's k field repeats C4's."""
    c4 = workloads.generate("C4", N=N)
    w1 = workloads.generate("C4w", N=N, param=1)
    for k in ("row_ptr", "col", "val", "b", "xstar"):
        assert np.array_equal(c4[k], w1[k])
    G = 3
    s = workloads.generate("C4w", N=N, param=G)
    Nz = G * N
    assert s["n"] == N * N * Nz and s["nnz"] == 7 * N * N * Nz - 4 * N * Nz - 2 * N * N
    cuts = [0, 7, s["n"] // 3, s["n"] // 3 + 1, s["n"]]
    parts = [workloads.generate_rows("C4w", a, b, N=N, param=G) for a, b in zip(cuts, cuts[1:])]
    off = np.cumsum([0] + [p["nnz"] for p in parts])
    rp = np.concatenate([[0]] + [p["row_ptr"][1:] + o for p, o in zip(parts, off)])
    assert np.array_equal(rp, s["row_ptr"])
    for k in ("col", "val", "b", "xstar"):
        assert np.array_equal(np.concatenate([p[k] for p in parts]), s[k])
    # the middle block's interior rows (planes 1..N-2) equal C4's
    NN = N * N
    b1 = workloads.generate_rows("C4w", N * NN + NN, 2 * N * NN - NN, N=N, param=G)
    ref = slice(c4["row_ptr"][NN], c4["row_ptr"][N * NN - NN])
    assert np.array_equal(b1["val"], c4["val"][ref])
    assert np.array_equal(b1["col"] - N * NN, c4["col"][ref])
