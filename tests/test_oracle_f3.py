"""Pins of the oracle's setup variants: true-IMPES column-sum
lumping (eq:CPR_CSL), the diagonal A_ps of step 4, the
fixed-stress modulus scale (remark P:443) and the row-sum-lumping fixed-stress
diagonal (eq:FS_RSL) -- against a hand-worked example, special cases
that reduce to the default path, and a dense solve of the RSL definition.  CPU only."""
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden", "cpr_2cell.txt")


def _two_cell(aps_offdiag=True):
    """nx=2, ny=nz=1: A_uu = I (decoupled mechanics), A_uf = A_fu = 0, A_ff from the fixture."""
    blocks, fs, rows = {}, np.zeros((2, 2)), []
    for line in open(GOLD):
        t = line.split()
        if not t or t[0].startswith("#"):
            continue
        if t[0] == "block":
            blocks[(int(t[1]), int(t[2]))] = np.array([float(x) for x in t[3:7]]).reshape(2, 2)
        elif t[0] == "fs":
            fs[int(t[1])] = [float(t[2]), float(t[3])]
        else:
            rows.append((t[0], float(t[1]), [float(x) for x in t[2:]]))
    if not aps_offdiag:
        for k in ((0, 1), (1, 0)):
            blocks[k] = blocks[k].copy(); blocks[k][1, 0] = 0.0
    nx, ny, nz = 2, 1, 1
    Nn = 12
    uu_val = np.tile(np.eye(3), (Nn, 1, 1))
    ff_val = np.array([blocks[(0, 0)], blocks[(0, 1)], blocks[(1, 0)], blocks[(1, 1)]])
    pb = synth.Problem(nx=nx, ny=ny, nz=nz, params={},
                       uu_rowptr=np.arange(Nn + 1, dtype=np.int32), uu_col=np.arange(Nn, dtype=np.int32), uu_val=uu_val,
                       uf_rowptr=np.zeros(Nn + 1, np.int32), uf_col=np.zeros(0, np.int32), uf_val=np.zeros((0, 3, 2)),
                       fu_rowptr=np.zeros(3, np.int32), fu_col=np.zeros(0, np.int32), fu_val=np.zeros((0, 2, 3)),
                       ff_rowptr=np.array([0, 2, 4], np.int32), ff_col=np.array([0, 1, 0, 1], np.int32), ff_val=ff_val,
                       fs=fs, x_rand=np.zeros(3 * Nn + 4), b=np.ones(3 * Nn + 4))
    return pb, rows


@pytest.mark.parametrize("row", [0, 1, 2])
def test_cpr_two_cell_hand_values(row):
    """D_ss, D_ps and S_pp of the hand-worked two-cell example (fixture cites the passages)."""
    pb, rows = _two_cell()
    mode, scale, vals = rows[row]
    o = oracle.Oracle(pb, cpr_mode=int(mode == "true"), fs_modulus_scale=scale).setup()
    Dss, Dps, fs_eff = o.cpr()
    _, rp, ci, v = o.spp()
    assert np.allclose(Dss, vals[0:2], rtol=0, atol=1e-15)
    assert np.allclose(Dps, vals[2:4], rtol=0, atol=1e-15)
    assert np.allclose(fs_eff, pb.fs / scale, rtol=0, atol=0)
    assert list(rp) == [0, 2, 4] and list(ci) == [0, 1, 0, 1]
    assert np.allclose(v, vals[4:8], rtol=0, atol=1e-14)


def test_true_equals_quasi_without_off_diagonal_coupling():
    """With no off-diagonal A_ss / A_ps entries the column sums ARE the diagonals (eq:CPR_CSL = P:575)."""
    pb = synth.generate("C1")
    ff = pb.ff_val.copy()
    diag = np.zeros(len(pb.ff_col), bool)
    for i in range(pb.Nc):
        for q in range(pb.ff_rowptr[i], pb.ff_rowptr[i + 1]):
            diag[q] = pb.ff_col[q] == i
    ff[~diag, 0, 0] = 0.0
    ff[~diag, 1, 0] = 0.0
    pb.ff_val = ff
    a = oracle.Oracle(pb, cpr_mode=0).setup()
    b = oracle.Oracle(pb, cpr_mode=1).setup()
    for x, y in zip(a.cpr()[:2] + (a.spp()[3],), b.cpr()[:2] + (b.spp()[3],)):
        assert np.array_equal(x, y)


def test_true_impes_column_sums_match_transpose():
    """D = diag(A^T e) (eq:CPR_CSL) = scipy's column sums of the scalar A_ss, A_ps (sum order aside)."""
    pb = synth.generate("C1")
    o = oracle.Oracle(pb, cpr_mode=1).setup()
    Dss, Dps, _ = o.cpr()
    _, (_, _, _, Aff) = synth.to_scipy(pb)
    Aff = Aff.toarray()
    assert np.allclose(Dss, Aff[0::2, 0::2].sum(axis=0), rtol=1e-13, atol=0)
    assert np.allclose(Dps, Aff[1::2, 0::2].sum(axis=0), rtol=1e-13, atol=1e-300)
    qi = oracle.Oracle(pb, cpr_mode=0).setup().cpr()
    assert not np.array_equal(Dss, qi[0])        # the reductions differ on a coupled problem


def test_diag_aps_equals_full_when_aps_is_diagonal():
    """Step 4 with D_ps^(CPR) = with the full A_ps when A_ps has no off-diagonal entries."""
    pb, _ = _two_cell(aps_offdiag=False)
    v = np.random.default_rng(5).uniform(-1, 1, pb.n)
    za = oracle.Oracle(pb, aps_mode=0).setup().apply(v)
    zb = oracle.Oracle(pb, aps_mode=1).setup().apply(v)
    assert np.allclose(za, zb, rtol=0, atol=1e-15 * np.abs(za).max())
    pb2 = synth.generate("C1")              # coupled A_ps: the two steps 4 differ (the 2-cell ILU is exact)
    v2 = np.random.default_rng(5).uniform(-1, 1, pb2.n)
    zc = oracle.Oracle(pb2, aps_mode=0).setup().apply(v2)
    zd = oracle.Oracle(pb2, aps_mode=1).setup().apply(v2)
    assert np.abs(zc - zd).max() > 1e-12 * np.abs(zc).max()


def test_modulus_scale_is_a_scaled_fs_input():
    """fs_modulus_scale = 4 (K_dr -> 4 K_dr) is exactly the default path with D_fs / 4 given (power of two)."""
    pb = synth.generate("C1")
    a = oracle.Oracle(pb, fs_modulus_scale=4.0).setup()
    pb4 = synth.generate("C1"); pb4.fs = pb4.fs / 4.0
    b = oracle.Oracle(pb4).setup()
    assert np.array_equal(a.spp()[3], b.spp()[3])
    assert np.array_equal(a.apply(pb.b), b.apply(pb.b))


def test_rsl_exact_solve_matches_dense_definition():
    """eq:FS_RSL with an exact A_uu solve (mech_mode 1, one Richardson step = A_uu^-1 g):
    D_sp = -diag(A_su A_uu^-1 A_up e), D_pp = -diag(A_pu A_uu^-1 A_up e), by numpy.linalg.solve."""
    pb = synth.generate("C1")
    o = oracle.Oracle(pb, fs_mode=1, rsl_iters=1, mech_mode=1).setup()
    _, _, fs = o.cpr()
    _, (Auu, Auf, Afu, _) = synth.to_scipy(pb)
    Auu, Auf, Afu = Auu.toarray(), Auf.toarray(), Afu.toarray()
    g = Auf[:, 1::2].sum(axis=1)                  # A_up e
    y = np.linalg.solve(Auu, g)
    ref = np.stack([-(Afu[0::2] @ y), -(Afu[1::2] @ y)], axis=1)
    assert np.allclose(fs, ref, rtol=1e-9, atol=1e-12 * np.abs(ref).max())


def test_rsl_richardson_converges_to_the_definition():
    """With the AMG preconditioner, more Richardson steps approach the exact RSL diagonal."""
    pb = synth.generate("C1")
    exact = oracle.Oracle(pb, fs_mode=1, rsl_iters=1, mech_mode=1).setup().cpr()[2]
    errs = []
    for k in (1, 4, 40):
        fs = oracle.Oracle(pb, fs_mode=1, rsl_iters=k).setup().cpr()[2]
        errs.append(np.abs(fs - exact).max() / np.abs(exact).max())
    assert errs[2] < errs[1] < errs[0] and errs[2] < 1e-2, errs


@pytest.mark.parametrize("opts", [dict(cpr_mode=1), dict(aps_mode=1), dict(fs_mode=1), dict(fs_modulus_scale=2.0),
                                  dict(cpr_mode=1, aps_mode=1)])
def test_variants_converge(opts):
    """Every variant still gives a convergent FGMRES (rtol 1e-8, true residual) on C1."""
    pb = synth.generate("C1")
    o = oracle.Oracle(pb, **opts).setup()
    x, info = o.solve(pb.b, rtol=1e-8, m=64)
    assert info["status"] == 0 and info["true_relres"] <= 1e-8


# ---------------------------------------------------------------- NEXT-f2: second stage
def _tile_lower(pb, tile):
    """Dense block-lower-triangular part (incl. diagonal blocks) of A_ff restricted to tile-local couplings."""
    import scipy.sparse as sp
    n2 = 2 * pb.Nc
    A = sp.bsr_matrix((pb.ff_val, pb.ff_col, pb.ff_rowptr), shape=(n2, n2)).toarray()

    def tile_of(c):
        i, j, k = c % pb.nx, (c // pb.nx) % pb.ny, c // (pb.nx * pb.ny)
        return (i // tile[0], j // tile[1], k // tile[2])

    L = np.zeros_like(A)
    for K in range(pb.Nc):
        for J in range(K + 1):
            if tile_of(K) == tile_of(J):
                L[2 * K:2 * K + 2, 2 * J:2 * J + 2] = A[2 * K:2 * K + 2, 2 * J:2 * J + 2]
    return A, L


def test_bgs_sweep_is_tile_block_forward_substitution():
    """One hybrid block GS sweep from zero = (L + D)^-1 w with L + D the tile-local block-lower triangle in
    natural order (R-hbgs); checked with a dense solve of that block-lower matrix (its 2x2 diagonal blocks
    are full, so it is block- not scalar-triangular)."""
    pb = synth.generate(nx=4, ny=3, nz=4, recipe=2, perm_sigma=2.0)
    tile = (2, 3, 2)
    A, L = _tile_lower(pb, tile)
    w = np.random.default_rng(9).uniform(-1, 1, 2 * pb.Nc)
    got = oracle.Bgs(pb.nx, pb.ny, pb.nz, tile, pb.ff_rowptr, pb.ff_col, pb.ff_val).apply(w)
    ref = np.linalg.solve(L, w)
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)


def test_second_stage_sweeps_converge_to_the_local_solve():
    """Steps 6-8 repeated (local_sweeps) with the block-GS or ILU second stage and no first stage acting on f
    (A_uf = A_fu = 0, b_u = 0, exact pressure AMG replaced by the dense solve) drive the flow residual down
    monotonically: block GS / ILU are convergent splittings of the (diagonally dominant) S_ff^FS."""
    pb = synth.generate("C1")
    pb.uf_val[:] = 0.0; pb.fu_val[:] = 0.0
    nu = 3 * pb.Nn
    v = np.zeros(pb.n); v[nu:] = np.random.default_rng(2).uniform(-1, 1, pb.n - nu)
    import scipy.sparse as sp
    n2 = 2 * pb.Nc
    S = sp.bsr_matrix((pb.ff_val, pb.ff_col, pb.ff_rowptr), shape=(n2, n2)).toarray()
    S[0::2, 1::2] += np.diag(pb.fs[:, 0]); S[1::2, 1::2] += np.diag(pb.fs[:, 1])
    for stage in (0, 1):
        res = []
        for k in (1, 2, 4, 8):
            z = oracle.Oracle(pb, second_stage=stage, local_sweeps=k, pres_mode=1).setup().apply(v)
            res.append(np.linalg.norm(v[nu:] - S @ z[nu:]) / np.linalg.norm(v[nu:]))
        assert all(b < a for a, b in zip(res, res[1:])), (stage, res)


def test_one_sweep_ilu_is_the_default_path():
    """second_stage 0 with local_sweeps 1 is bitwise the default Algorithm 1."""
    pb = synth.generate("C1")
    a = oracle.Oracle(pb).setup().apply(pb.b)
    b = oracle.Oracle(pb, second_stage=0, local_sweeps=1).setup().apply(pb.b)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("opts", [dict(second_stage=1, local_sweeps=3), dict(second_stage=0, local_sweeps=2)])
def test_second_stage_variants_converge(opts):
    pb = synth.generate("C1")
    x, info = oracle.Oracle(pb, **opts).setup().solve(pb.b, rtol=1e-8, m=64)
    assert info["status"] == 0 and info["true_relres"] <= 1e-8


# ---------------------------------------------------------------- NEXT-f4 (iii): sequential (Richardson) embedding
def test_richardson_embedding_exact_and_decoupled():
    """Remark P:640-642: x <- x + M^-1 (b - A x).  With A_uf = A_fu = 0 and exact sub-solves M^-1 = A^-1, so one
    step solves the system; with the coupling and an exact mechanics solve it is the fixed-stress sequential
    scheme, a contraction: it converges to the dense solution."""
    import scipy.sparse as sp
    pb = synth.generate("C1")
    o = oracle.Oracle(pb, mech_mode=1).setup()
    x, info = o.richardson(pb.b, rtol=1e-8, maxit=1000)
    A, _ = synth.to_scipy(pb)
    assert info["status"] == 0 and info["true_relres"] <= 1e-8
    assert np.linalg.norm(x - pb.x_rand) <= 1e-4 * np.linalg.norm(pb.x_rand)   # cond(A) ~ 1e4 at rtol 1e-8
    pb.uf_val[:] = 0.0; pb.fu_val[:] = 0.0
    A, _ = synth.to_scipy(pb)
    b = A @ pb.x_rand
    o2 = oracle.Oracle(pb, mech_mode=1, ff_mode=1).setup()
    x2, info2 = o2.richardson(b, rtol=1e-8, maxit=10)
    assert info2["iterations"] == 1 and info2["true_relres"] <= 1e-10


def test_richardson_steps_and_contraction_on_the_staircase():
    """Remark P:640-642 with the paper's stages (one SDC V-cycle, CPR, tile ILU): every step is
    x + M^-1 (b - A x) assembled from the operator and the preconditioner application (checked against the scipy
    matrix), the reported residual is the true one, and on the staircase ST0 the iteration contracts (52 steps to
    1e-6) while FGMRES with the same preconditioner needs fewer applications (the remark's "superior")."""
    pb = synth.generate("ST0")
    A, _ = synth.to_scipy(pb)
    o = oracle.Oracle(pb).setup()
    x3, i3 = o.richardson(pb.b, rtol=1e-30, maxit=3)
    x = np.zeros(pb.n)
    for _ in range(3):
        x = x + o.apply(pb.b - A @ x)
    assert i3["iterations"] == 3
    assert np.linalg.norm(x3 - x) <= 1e-12 * np.linalg.norm(x)
    assert abs(i3["true_relres"] - np.linalg.norm(pb.b - A @ x3) / np.linalg.norm(pb.b)) <= 1e-10 * i3["true_relres"]
    hist = [o.richardson(pb.b, rtol=1e-30, maxit=k)[1]["true_relres"] for k in (4, 8, 16, 32)]
    assert all(b < a for a, b in zip(hist, hist[1:])) and hist[-1] < 1e-4
    xr, ir = o.richardson(pb.b, rtol=1e-6, maxit=400)
    xk, ik = o.solve(pb.b, rtol=1e-6, m=64)
    assert ir["status"] == 0 and ik["status"] == 0 and ik["iterations"] < ir["iterations"]
