"""Soft-error semantics of the setup (SPEC S:394 coarsening stagnation -> direct solve, S:403 zero D_ss ->
skip + diagnostic, S:421 singular pivot -> perturb + diagnostic) and SPEC's smoothing special case,
pinned on the oracle against closed forms.  The same inputs are run through the CUDA path in
tests/test_gpu_soft.py.  CPU only."""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle
import synth


def zero_dss_problem(cell=4, **kw):
    """A generated problem whose A_ss diagonal entry of `cell` is zeroed (D_ss,cell = 0)."""
    pb = synth.generate(**(kw or dict(nx=3, ny=3, nz=3, recipe=2, perm_sigma=2.0)))
    pb.ff_val = pb.ff_val.copy()
    q = pb.ff_rowptr[cell] + int(np.flatnonzero(pb.ff_col[pb.ff_rowptr[cell]:pb.ff_rowptr[cell + 1]] == cell)[0])
    pb.ff_val[q, 0, 0] = 0.0
    return pb, q


def singular_pivot_problem(cell=0, **kw):
    """A generated problem whose fixed-stress diagonal block S^FS_KK of `cell` (the first cell of its ILU tile,
    so U_KK = S^FS_KK) has two equal columns: A_sp + D_sp := A_ss, A_pp + D_pp := A_ps."""
    pb = synth.generate(**(kw or dict(nx=3, ny=3, nz=3, recipe=2, perm_sigma=2.0)))
    pb.ff_val = pb.ff_val.copy()
    q = pb.ff_rowptr[cell] + int(np.flatnonzero(pb.ff_col[pb.ff_rowptr[cell]:pb.ff_rowptr[cell + 1]] == cell)[0])
    B = pb.ff_val[q]
    B[0, 1] = B[0, 0] - pb.fs[cell, 0]
    B[1, 1] = B[1, 0] - pb.fs[cell, 1]
    return pb, q


def stagnating_problem(nz=80):
    """1 x 2 x nz cells with z-blocks of ONE cell plane: level 0 aggregates each plane into (at most) one
    aggregate, the next level has no same-z-block coupling at all (every row isolated, no aggregate) and more
    than 64 rows, so both hierarchies stop there with a dense solve."""
    return synth.generate(nx=1, ny=2, nz=nz, recipe=2, perm_sigma=1.0), dict(zblock=1)


def test_zero_dss_row_is_skipped_and_counted():
    """D_ss,i = 0: z_s,i = 0 and S_pp row i = A_pp^FS row i (no correction), counted once.
    Checked against the dense M_G of eq:S1_prec with D_ss^-1 replaced by 0 on that row."""
    cell = 4
    pb, _ = zero_dss_problem(cell)
    o = oracle.Oracle(pb, mech_mode=1, pres_mode=1, local_mode=2).setup()
    assert o.counters()["skipped_dss"] == 1
    A, (Auu, Auf, Afu, Aff) = synth.to_scipy(pb)
    Auu, Afu, Aff = Auu.toarray(), Afu.toarray(), Aff.toarray()
    Sfs = Aff.copy()
    Sfs[0::2, 1::2] += np.diag(pb.fs[:, 0])
    Sfs[1::2, 1::2] += np.diag(pb.fs[:, 1])
    nc = pb.Nc
    Ass, Aps = Aff[0::2, 0::2], Aff[1::2, 0::2]
    dss, dps = np.diag(Ass).copy(), np.diag(Aps)
    assert dss[cell] == 0.0
    dinv = np.where(dss != 0.0, 1.0 / np.where(dss != 0.0, dss, 1.0), 0.0)
    Spp = Sfs[1::2, 1::2] - np.diag(dps * dinv) @ Sfs[0::2, 1::2]
    np.testing.assert_array_equal(Spp[cell], Sfs[1::2, 1::2][cell])
    Dss_rp, rp, ci, v = o.spp()
    got = sp.csr_matrix((v, ci, rp), shape=(nc, nc)).toarray()
    assert np.abs(got - Spp).max() <= 1e-13 * np.abs(Spp).max()
    MG = np.block([[np.eye(nc), np.zeros((nc, nc))], [np.zeros((nc, nc)), np.linalg.inv(Spp)]]) \
        @ np.block([[np.eye(nc), np.zeros((nc, nc))], [-Aps, np.eye(nc)]]) \
        @ np.block([[np.diag(dinv), np.zeros((nc, nc))], [np.zeros((nc, nc)), np.eye(nc)]])
    v = np.random.default_rng(4).uniform(-1, 1, pb.n)
    z = o.apply(v)
    nu = 3 * pb.Nn
    yf = v[nu:] - Afu @ np.linalg.solve(Auu, v[:nu])
    zp = MG @ np.concatenate([yf[0::2], yf[1::2]])
    got = np.concatenate([z[nu:][0::2], z[nu:][1::2]])
    assert got[cell] == 0.0                                   # z_s of the skipped row
    assert np.linalg.norm(got - zp) <= 1e-8 * np.linalg.norm(zp)


def test_singular_ilu_pivot_is_perturbed_and_counted():
    """A singular U_KK is replaced by U_KK + 1e-12 max|U_KK| I and counted; the full setup counts it
    exactly once, and the preconditioner stays finite."""
    pb, q = singular_pivot_problem(0)
    o = oracle.Oracle(pb).setup()
    assert o.counters()["perturbed"] == 1
    z = o.apply(np.random.default_rng(5).uniform(-1, 1, pb.n))
    assert np.all(np.isfinite(z))


def test_singular_pivot_closed_form_on_one_cell():
    """One cell: the tile ILU(0) IS the perturbed block inverse, dz = (B + delta I)^-1 w, delta = 1e-12 max|B|."""
    B = np.array([[2.0, 4.0], [1.0, 2.0]])                   # rank one
    ilu = oracle.Ilu(1, 1, 1, (16, 16, 16), np.array([0, 1], np.int32), np.array([0], np.int32), B.reshape(1, 2, 2))
    w = np.array([0.3, -0.7])
    d = 1e-12 * 4.0
    ref = np.linalg.solve(B + d * np.eye(2), w)
    got = ilu.apply(w)
    assert np.abs(got - ref).max() <= 1e-6 * np.abs(ref).max()     # cond(B + delta I) ~ 1e12
    assert np.abs(got).max() > 1e10


def test_coarsening_stagnation_falls_back_to_a_dense_level():
    """S:394 / SURVEY D4: a level that yields no aggregate is solved densely, counted once per hierarchy; the
    cycle below the stagnated level is then the exact two-grid cycle."""
    pb, kw = stagnating_problem()
    o = oracle.Oracle(pb, **kw).setup()
    assert o.counters()["fallbacks"] == 2
    for which in (0, 1):
        H = o.hierarchy(which)
        assert H[-1]["coarsest"] and H[-1]["n"] > 64
    # standalone: the V-cycle equals (I - D^-1 A)(I - P A_c^-1 P^T A)(I - D^-1 A) with an exact coarse solve
    nx, ny, nz = 2, 2, 80
    n = nx * ny * nz
    A = _lap7(nx, ny, nz)
    zb = (np.arange(n) // (nx * ny)).astype(np.int32)
    amg = oracle.Amg(A.indptr, A.indices, A.data, zb)
    Ls = amg.levels()
    assert len(Ls) == 2 and Ls[1]["coarsest"] and Ls[1]["n"] == nz
    L0 = Ls[0]
    P = sp.csr_matrix((L0["P_v"][:, 0], L0["P_ci"], L0["P_rp"]), shape=(n, L0["nagg"])).toarray()
    Ad = A.toarray()
    S = np.eye(n) - Ad / np.abs(Ad).sum(1)[:, None]
    E_ref = S @ (np.eye(n) - P @ np.linalg.solve(P.T @ Ad @ P, P.T @ Ad)) @ S
    M = np.stack([amg.vcycle(e) for e in np.eye(n)], 1)
    assert np.abs(np.eye(n) - M @ Ad - E_ref).max() <= 1e-10


def test_stagnation_beyond_the_dense_limit_is_an_error():
    """D4: stagnation on a level of more than 4096 rows is an error, not a silent answer."""
    n = 4200
    A = sp.diags([-np.ones(n - 1), 2.5 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1]).tocsr()
    A.sort_indices()
    zb = np.arange(n, dtype=np.int32)                         # every row its own z-block: nothing aggregates
    with pytest.raises(RuntimeError):
        oracle.Amg(A.indptr, A.indices, A.data, zb)


def _lap7(nx, ny, nz):
    n = nx * ny * nz
    idx = np.arange(n).reshape(nz, ny, nx)
    rows, cols = [], []
    for d in ((1, 0, 0), (0, 1, 0), (0, 0, 1)):
        a = idx[:nz - d[2], :ny - d[1], :nx - d[0]].ravel()
        b = idx[d[2]:, d[1]:, d[0]:].ravel()
        rows += [a, b]
        cols += [b, a]
    r, c = np.concatenate(rows), np.concatenate(cols)
    A = sp.csr_matrix((-np.ones(len(r)), (r, c)), shape=(n, n)).tolil()
    A.setdiag(-np.asarray(A.sum(1)).ravel() + 0.01)
    A = A.tocsr()
    A.sort_indices()
    return A


def test_isolated_rows_are_solved_by_the_first_smoothing_step():
    """a diagonal row is solved exactly by one l1-Jacobi step.  Rows without off-diagonals (the
    Dirichlet rows of D11) are isolated (D2), get a zero P row, so the coarse correction and the post-smoothing
    leave x_i = b_i / a_ii; a purely diagonal matrix is solved exactly by the V-cycle."""
    A = _lap7(6, 5, 6).tolil()
    dirichlet = np.arange(0, 30)                              # bottom plane: identity rows, zero columns
    for i in dirichlet:
        A[i, :] = 0.0
        A[:, i] = 0.0
        A[i, i] = 3.0
    A = A.tocsr()
    A.eliminate_zeros()
    A.sort_indices()
    amg = oracle.Amg(A.indptr, A.indices, A.data, None, amg_coarse_max=8)
    assert len(amg.levels()) >= 2
    b = np.random.default_rng(9).uniform(-1, 1, A.shape[0])
    x = amg.vcycle(b)
    np.testing.assert_allclose(x[dirichlet], b[dirichlet] / 3.0, rtol=1e-15)
    D = sp.diags(np.linspace(1.0, 4.0, 200)).tocsr()
    D.sort_indices()
    amgd = oracle.Amg(D.indptr, D.indices, D.data, None)
    bd = np.random.default_rng(10).uniform(-1, 1, 200)
    np.testing.assert_allclose(amgd.vcycle(bd), bd / D.diagonal(), rtol=1e-15)
