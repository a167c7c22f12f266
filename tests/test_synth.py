"""Checks of the seeded input generator (synth/): it is shared by both sides, so
its structure is pinned here against the paper and against closed forms."""
import os

import numpy as np
import pytest

import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_dof_counts_match_paper_table2():
    """DoF of the paper's staircase meshes = sizes of our grids."""
    rows = [l.split() for l in open(os.path.join(GOLD, "staircase_dof.txt")) if l.strip() and not l.startswith("#")]
    for nx, ny, nz, dof in rows:
        assert synth.sizes(int(nx), int(ny), int(nz))["n"] == int(dof)


def test_block_counts_closed_form():
    s = synth.sizes(8, 8, 8)
    assert s["Buu"] == 25 ** 3 and s["Buf"] == 8 * 512 and s["Bff"] == 512 + 2 * 3 * 7 * 64


def test_rhs_is_A_times_xrand():
    pb = synth.generate("C1")
    A, _ = synth.to_scipy(pb)
    assert np.abs(A @ pb.x_rand - pb.b).max() <= 1e-12 * np.abs(pb.b).max()


def test_columns_sorted_unique():
    pb = synth.generate("C1")
    for rp, ci in ((pb.uu_rowptr, pb.uu_col), (pb.uf_rowptr, pb.uf_col), (pb.fu_rowptr, pb.fu_col), (pb.ff_rowptr, pb.ff_col)):
        for i in range(len(rp) - 1):
            c = ci[rp[i]:rp[i + 1]]
            assert np.all(np.diff(c) > 0)


def _rigid_modes(pb):
    nx, ny, nz = pb.nx, pb.ny, pb.nz
    h = pb.params["length"] / nx
    k, j, i = np.meshgrid(np.arange(nz + 1), np.arange(ny + 1), np.arange(nx + 1), indexing="ij")
    X = np.stack([i.ravel() * h, j.ravel() * h, k.ravel() * h], 1)
    modes = []
    for d in range(3):
        m = np.zeros_like(X); m[:, d] = 1; modes.append(m.ravel())
    for a, b in ((0, 1), (1, 2), (0, 2)):
        m = np.zeros_like(X); m[:, a] = -X[:, b]; m[:, b] = X[:, a]; modes.append(m.ravel())
    return modes


def test_rigid_body_modes_in_kernel_of_elasticity():
    """6 rigid motions span the kernel of the unconstrained Q1 stiffness; the
    gravity term also annihilates them (div u = 0).  SURVEY c.4."""
    pb = synth.generate(nx=3, ny=3, nz=3, recipe=1, dirichlet_bottom=0, row_scale=0)
    _, (Auu, *_r) = synth.to_scipy(pb)
    scale = abs(Auu).max()
    for r in _rigid_modes(pb):
        assert np.abs(Auu @ r).max() <= 1e-10 * scale * np.abs(r).max()
    # and exactly 6 zero eigenvalues
    ev = np.linalg.eigvals(Auu.toarray())
    assert np.sum(np.abs(ev) < 1e-9 * scale) == 6


def test_tpfa_pressure_rows_sum_to_zero():
    """g = 0, uniform state, incompressible fluids, no wells: every TPFA
    pressure-derivative row sums to zero."""
    pb = synth.generate(nx=4, ny=3, nz=5, recipe=1, gravity=0.0, c_w=0.0, c_nw=0.0, wells=0, row_scale=0, dirichlet_bottom=0)
    _, (_, _, _, Aff) = synth.to_scipy(pb)
    Aff = Aff.toarray()
    rows = Aff[:, 1::2].sum(1)
    assert np.abs(rows).max() <= 1e-12 * np.abs(Aff[:, 1::2]).max()
    # and the matrix is symmetric in its pressure couplings up to the phase weighting: off-diagonals <= 0
    App = Aff[1::2, 1::2]
    assert (App - np.diag(np.diag(App)) <= 0).all()


def test_decoupled_limit():
    """b = 0 and g = 0 => A_us = A_up = A_su = A_pu = 0."""
    pb = synth.generate(nx=3, ny=3, nz=3, recipe=1, biot=0.0, gravity=0.0)
    assert np.abs(pb.uf_val).max() == 0.0 and np.abs(pb.fu_val).max() == 0.0


def test_closed_form_couplings_on_cubes():
    """A_su[K,(a,d)] = s rho_w (+-h^2/4), unscaled, b = 1."""
    pb = synth.generate(nx=2, ny=2, nz=2, recipe=1, row_scale=0, dirichlet_bottom=0, p_unit=1.0)
    h = pb.params["length"] / 2
    s = pb.fields["sat"]; p = pb.fields["pres"]
    rw = 1035.0 * (1 + 4.34e-10 * (p - 1e7))
    for K in range(pb.Nc):
        blk = pb.fu_val[8 * K:8 * K + 8, 0, :]
        assert np.allclose(np.abs(blk), s[K] * rw[K] * h * h / 4, rtol=1e-13)
        assert np.allclose(blk.sum(0), 0.0, atol=1e-12 * s[K] * rw[K] * h * h)


def test_fixed_stress_hand_value():
    """D_sp = V b^2/K_dr s rho_w: V = 1, E = 5000 MPa, nu = 0.25, s = 0.5,
    rho_w = 1035 -> 0.15525 in per-MPa units."""
    Kdr = 5000.0 / (3 * (1 - 2 * 0.25))
    assert abs(1.0 * 1.0 / Kdr * 0.5 * 1035.0 - 0.15525) < 1e-12
    # the generator's D_sp, unscaled, matches the same formula cell by cell
    pb = synth.generate(nx=2, ny=2, nz=2, recipe=1, row_scale=0, p_unit=1.0)
    h = pb.params["length"] / 2
    Kdr = pb.fields["E"] / (3 * (1 - 2 * 0.25))
    rw = 1035.0 * (1 + 4.34e-10 * (pb.fields["pres"] - 1e7))
    np.testing.assert_allclose(pb.fs[:, 0], h ** 3 / Kdr * pb.fields["sat"] * rw, rtol=1e-14)


def test_dirichlet_rows_identity():
    pb = synth.generate("C1")
    nb = (pb.nx + 1) * (pb.ny + 1)
    for n in range(nb):
        for q in range(pb.uu_rowptr[n], pb.uu_rowptr[n + 1]):
            want = np.eye(3) if pb.uu_col[q] == n else np.zeros((3, 3))
            assert np.array_equal(pb.uu_val[q], want)
    assert np.abs(pb.uf_val[pb.uf_rowptr[0]:pb.uf_rowptr[nb]]).max() == 0


def test_seeded_reproducible():
    a = synth.generate("C1"); b = synth.generate("C1")
    assert np.array_equal(a.uu_val, b.uu_val) and np.array_equal(a.b, b.b)
    c = synth.generate("C1", seed=1)
    assert not np.array_equal(a.x_rand, c.x_rand)
