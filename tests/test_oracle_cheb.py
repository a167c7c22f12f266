"""Pins of the oracle's Chebyshev AMG smoother (tsp_options / orc_opts amg_smoother = 2; north_star "fused
Jacobi/Chebyshev or l1-Jacobi AMG smoothers"; reading R-cheb in DESIGN.md).  The smoother is
`degree` steps of the Chebyshev iteration (Saad, Alg. 12.1) for D_l1^-1 A x = D_l1^-1 b on [lower, 1].  The pins
check it against what the mathematics fixes, independently of the iteration's recurrences:
  * the error after m steps is p_m(D^-1 A) e_0 with p_m(t) = T_m((theta - t)/delta) / T_m(theta/delta) -- evaluated
    here from an eigendecomposition and numpy's Chebyshev-series evaluation (Clenshaw), not from the iteration;
  * degree 1 is damped Jacobi with omega = 1/theta;
  * the V-cycle with Chebyshev pre- and post-smoothing is a symmetric operator for SPD input and contracts the
    error on a 3D Poisson problem;
  * sign equivariance through the signed l1 diagonal (R-l1).
CPU only."""
import numpy as np
import pytest
import scipy.sparse as sp
from numpy.polynomial import chebyshev as npc

import oracle
import synth


def _variable_poisson_2d(n, seed):
    """SPD 5-point operator with random positive face coefficients (heterogeneous diffusion)."""
    rng = np.random.default_rng(seed)
    N = n * n
    rows, cols, vals = [], [], []
    diag = np.full(N, 1e-3)
    for j in range(n):
        for i in range(n):
            k = i + n * j
            for di, dj in ((1, 0), (0, 1)):
                if i + di < n and j + dj < n:
                    m = (i + di) + n * (j + dj)
                    w = np.exp(rng.normal())
                    rows += [k, m]; cols += [m, k]; vals += [-w, -w]
                    diag[k] += w; diag[m] += w
    A = sp.csr_matrix((vals + list(diag), (rows + list(range(N)), cols + list(range(N)))), shape=(N, N))
    A.sort_indices()
    return A


def _poly_error(A, lower, m):
    """p_m(D^-1 A) for the Chebyshev iteration on [lower, 1] (dense), through the eigendecomposition of the
    symmetric D^-1/2 A D^-1/2 and numpy's Chebyshev-series evaluation."""
    Ad = A.toarray()
    d = np.abs(Ad).sum(axis=1)                       # l1 diagonal (all diagonals positive here)
    s = 1.0 / np.sqrt(d)
    S = s[:, None] * Ad * s[None, :]
    lam, Q = np.linalg.eigh(S)
    a, b = lower, 1.0
    theta, delta = (a + b) / 2, (b - a) / 2
    Tm = np.zeros(m + 1); Tm[m] = 1.0
    p = npc.chebval((theta - lam) / delta, Tm) / npc.chebval(theta / delta, Tm)
    P_sym = (Q * p) @ Q.T
    return (s[:, None] * P_sym) / s[None, :]         # D^-1/2 p(S) D^1/2


@pytest.mark.parametrize("m", [1, 2, 3, 4])
@pytest.mark.parametrize("lower", [0.1, 0.3])
def test_error_is_the_chebyshev_polynomial(m, lower):
    A = _variable_poisson_2d(7, seed=m)
    rng = np.random.default_rng(10 + m)
    b = rng.uniform(-1, 1, A.shape[0])
    x0 = rng.uniform(-1, 1, A.shape[0])
    xs = np.linalg.solve(A.toarray(), b)
    E = _poly_error(A, lower, m)
    for start in (x0, None):
        e0 = xs - (start if start is not None else 0.0)
        want = xs - E @ e0
        got = oracle.cheb_smooth(A.indptr, A.indices, A.data, b, x0=start, degree=m, lower=lower)
        assert np.linalg.norm(got - want) <= 1e-11 * np.linalg.norm(want), (m, lower)


def test_degree_one_is_damped_jacobi():
    A = _variable_poisson_2d(6, seed=3)
    rng = np.random.default_rng(4)
    b, x0 = rng.uniform(-1, 1, A.shape[0]), rng.uniform(-1, 1, A.shape[0])
    d = np.abs(A.toarray()).sum(axis=1)
    theta = (0.3 + 1.0) / 2
    want = x0 + (b - A @ x0) / d / theta
    got = oracle.cheb_smooth(A.indptr, A.indices, A.data, b, x0=x0, degree=1, lower=0.3)
    assert np.allclose(got, want, rtol=1e-14, atol=1e-14)


def test_bad_parameters_are_refused():
    A = _variable_poisson_2d(3, seed=0)
    with pytest.raises(ValueError):
        oracle.cheb_smooth(A.indptr, A.indices, A.data, np.ones(9), degree=0)
    with pytest.raises(ValueError):
        oracle.cheb_smooth(A.indptr, A.indices, A.data, np.ones(9), lower=1.0)


def _poisson3d(n):
    I = sp.identity(n)
    T = sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1])
    A = (sp.kron(sp.kron(T, I), I) + sp.kron(sp.kron(I, T), I) + sp.kron(sp.kron(I, I), T)).tocsr()
    A.sort_indices()
    return A


def test_vcycle_is_symmetric_and_contracts():
    A = _poisson3d(12)
    H = oracle.Amg(A.indptr, A.indices, A.data, amg_smoother=2)
    assert len(H.levels()) >= 3
    rng = np.random.default_rng(7)
    u, w = rng.uniform(-1, 1, A.shape[0]), rng.uniform(-1, 1, A.shape[0])
    Mu, Mw = H.vcycle(u), H.vcycle(w)
    assert abs(Mu @ w - u @ Mw) <= 1e-12 * abs(Mu @ w)
    # stationary V-cycle iteration: error reduction per cycle
    xs = rng.uniform(-1, 1, A.shape[0])
    b = A @ xs
    x = np.zeros_like(b)
    errs = []
    for _ in range(6):
        x = x + H.vcycle(b - A @ x)
        errs.append(np.linalg.norm(x - xs))
    assert errs[-1] / errs[-2] <= 0.35, errs
    # and a higher degree smooths better on the same hierarchy
    H3 = oracle.Amg(A.indptr, A.indices, A.data, amg_smoother=2, amg_cheb_degree=3)
    x3 = np.zeros_like(b)
    for _ in range(6):
        x3 = x3 + H3.vcycle(b - A @ x3)
    assert np.linalg.norm(x3 - xs) < errs[-1]


def test_sign_equivariance():
    """Signed l1 diagonal (R-l1): D(-A) = -D(A), so the smoother and the V-cycle of -A are minus those of A."""
    A = _variable_poisson_2d(8, seed=5)
    b = np.random.default_rng(8).uniform(-1, 1, A.shape[0])
    x1 = oracle.cheb_smooth(A.indptr, A.indices, A.data, b, degree=3)
    x2 = oracle.cheb_smooth(A.indptr, A.indices, -A.data, b, degree=3)
    assert np.array_equal(x1, -x2)
    H1 = oracle.Amg(A.indptr, A.indices, A.data, amg_smoother=2)
    H2 = oracle.Amg(A.indptr, A.indices, -A.data, amg_smoother=2)
    assert np.allclose(H1.vcycle(b), -H2.vcycle(b), rtol=0, atol=1e-13 * np.abs(H1.vcycle(b)).max())


def test_fgmres_with_chebyshev_smoothers_converges():
    pb = synth.generate("C1")
    x, info = oracle.Oracle(pb, amg_smoother=2).setup().solve(pb.b, rtol=1e-8)
    assert info["status"] == 0 and info["true_relres"] <= 1e-8
    _, info0 = oracle.Oracle(pb).setup().solve(pb.b, rtol=1e-8)
    assert info["iterations"] <= info0["iterations"] + 5, (info["iterations"], info0["iterations"])
