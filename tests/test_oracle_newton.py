"""Pins of the nonlinear residual (oracle/residual.c, Appendix B.1) -- CPU only.

The residual and the Jacobian come from two independent codes: residual.c and the CPU assembler of synth/
(itself pinned by tests/test_synth.py against closed forms, the paper's DoF counts and the rigid-body kernel).
Pinned here against what the mathematics fixes:
  * at u = 0 the Jacobian IS the derivative of the residual: central finite differences along random directions
    reproduce J dx row block by row block (momentum, water, non-wetting) to 1e-6 -- a dropped term, a wrong sign
    or a transposed index in either code fails it;
  * the residual is linear in u where the physics is (strain-free rows) and vanishes in a hydrostatic, well-free,
    single-phase state of the flow rows;
  * mass conservation: the flux terms of all cells sum to zero (the face contributions cancel in pairs), so the sum
    of the mass rows is the accumulation minus dt times the well terms.
"""
import numpy as np
import pytest

import oracle
import synth


def _state(cfg, **kw):
    f = synth.fields(cfg, x_rand=False, **kw)
    prm = f["params"]
    pb = synth.generate(cfg, **kw)
    s = synth.sizes(prm["nx"], prm["ny"], prm["nz"])
    x = np.zeros(s["n"])
    x[3 * s["Nn"]::2] = f["sat"]
    x[3 * s["Nn"] + 1::2] = f["pres"]
    fl = dict(E=f["E"], perm=f["perm"], phi0=f["phi"], pref=f["pres"], well=f["well"])
    return prm, fl, x, pb, s


def _raw_jacobian(pb, s, prm):
    """synth's blocks with the row scaling and the pressure unit undone (Dirichlet rows / columns marked)."""
    A, _ = synth.to_scipy(pb)
    A = A.tolil().tocsr()
    Nn, Nc = s["Nn"], s["Nc"]
    su, ss, sp = pb.scales
    rs = np.concatenate([np.full(3 * Nn, su), np.tile([ss, sp], Nc)])
    cs = np.concatenate([np.ones(3 * Nn), np.tile([1.0, prm["p_unit"]], Nc)])
    import scipy.sparse as sp_
    return sp_.diags(1.0 / rs) @ A @ sp_.diags(1.0 / cs)


def _direction(s, prm, rng, du=1e-3, ds=1e-2, dp=1e4):
    Nn, Nc = s["Nn"], s["Nc"]
    d = np.zeros(s["n"])
    d[:3 * Nn] = du * rng.uniform(-1, 1, 3 * Nn)
    nbot = (prm["nx"] + 1) * (prm["ny"] + 1)
    d[:3 * nbot] = 0.0                               # Dirichlet nodes stay fixed
    d[3 * Nn::2] = ds * rng.uniform(-1, 1, Nc)
    d[3 * Nn + 1::2] = dp * rng.uniform(-1, 1, Nc)
    return d


# state_dp != 0: a pressure gradient on every horizontal face, so no face sits exactly at the upwinding switch
# (Phi = 0, where the flux has a kink and central differences straddle it)
@pytest.mark.parametrize("cfg,kw", [("C1", dict(state_dp=1e6)),
                                    (None, dict(nx=6, ny=5, nz=7, recipe=2, perm_sigma=2.0, state_dp=2e6)),
                                    ("ST0", dict(nx=8, ny=8, nz=8, state_dp=1e6)),
                                    ("S10", dict(nx=5, ny=6, nz=12, burden=3, state_dp=1e6))])
def test_jacobian_is_the_derivative_of_the_residual(cfg, kw):
    prm, fl, x, pb, s = _state(cfg, **kw)
    J = _raw_jacobian(pb, s, prm)
    mprev = oracle.masses(prm, fl, x)
    dt = prm["dt"]
    rng = np.random.default_rng(7)
    Nn = s["Nn"]
    nbot = (prm["nx"] + 1) * (prm["ny"] + 1)
    rows = {"u": slice(3 * nbot, 3 * Nn), "w": slice(3 * Nn, None, 2), "nw": slice(3 * Nn + 1, None, 2)}
    for trial in range(3):
        d = _direction(s, prm, rng)
        eps = 1e-3
        fd = (oracle.residual(prm, fl, x + eps * d, mprev, dt) - oracle.residual(prm, fl, x - eps * d, mprev, dt)) / (2 * eps)
        Jd = J @ d
        for name, sl in rows.items():
            err = np.linalg.norm(fd[sl] - Jd[sl]) / np.linalg.norm(Jd[sl])
            assert err <= 1e-6, (cfg, trial, name, err)


def test_mechanics_rows_are_affine_in_u():
    """At fixed (s, p) the momentum residual is affine in u: r(x + d_u) - r(x) = J_uu d_u exactly (up to rounding),
    including the gravity term's strain part."""
    prm, fl, x, pb, s = _state("C1")
    J = _raw_jacobian(pb, s, prm)
    mprev = oracle.masses(prm, fl, x)
    d = _direction(s, prm, np.random.default_rng(3), ds=0.0, dp=0.0)
    r1, r0 = oracle.residual(prm, fl, x + d, mprev, prm["dt"]), oracle.residual(prm, fl, x, mprev, prm["dt"])
    Nn = s["Nn"]
    Jd = J @ d
    assert np.linalg.norm((r1 - r0)[:3 * Nn] - Jd[:3 * Nn]) <= 1e-10 * np.linalg.norm(Jd[:3 * Nn])


def test_discrete_hydrostatic_equilibrium_is_at_rest():
    """Water only (s = 1 - snwr: the non-wetting phase immobile), no wells, x at the previous masses, and the
    pressure in DISCRETE hydrostatic equilibrium of eq:num_flux_approx with the averaged compressible density
    (p_below = p_above + g h (rho_w(p_above) + rho_w(p_below)) / 2, solved per layer): every water flux vanishes,
    so the water rows are zero to rounding -- against the same state with the incompressible hydrostatic profile,
    which over the 10 km column (1e8 Pa) is NOT at rest."""
    prm, fl, x, pb, s = _state("C1")
    Nn, Nc = s["Nn"], s["Nc"]
    nx, ny, nz = prm["nx"], prm["ny"], prm["nz"]
    h, g = prm["length"] / nx, prm["gravity"]
    rho = lambda p: prm["rho_w0"] * (1 + prm["c_w"] * (p - prm["p0"]))   # noqa: E731
    layers = np.empty(nz)
    layers[nz - 1] = prm["p0"] + rho(prm["p0"]) * g * h / 2
    for k in range(nz - 2, -1, -1):
        pk = layers[k + 1]
        for _ in range(60):
            pk = layers[k + 1] + g * h * 0.5 * (rho(layers[k + 1]) + rho(pk))
        layers[k] = pk
    x = x.copy()
    x[3 * Nn::2] = 1.0 - prm["snwr"]
    x[3 * Nn + 1::2] = np.repeat(layers, nx * ny)
    fl = dict(fl, well=None)
    mprev = oracle.masses(prm, fl, x)
    R = oracle.residual(prm, fl, x, mprev, prm["dt"])
    x2 = x.copy()
    x2[3 * Nn + 1::2] = prm["p0"] + prm["rho_w0"] * g * (nz * h - (np.arange(Nc) // (nx * ny) + 0.5) * h)
    R2 = oracle.residual(prm, fl, x2, oracle.masses(prm, fl, x2), prm["dt"])
    assert np.abs(R2[3 * Nn::2]).max() > 1e3                  # the incompressible profile drives a flow
    assert np.abs(R[3 * Nn::2]).max() <= 1e-9 * np.abs(R2[3 * Nn::2]).max()


def test_fluxes_conserve_mass():
    prm, fl, x, pb, s = _state(None, nx=6, ny=5, nz=7, recipe=2, perm_sigma=2.0, state_dp=2e6)
    Nn = s["Nn"]
    fl0 = dict(fl, well=None)
    mprev = oracle.masses(prm, fl0, x)
    R = oracle.residual(prm, fl0, x, mprev, prm["dt"])
    # no wells, x at mprev: only the flux terms remain, and they cancel in pairs
    for ph in (0, 1):
        r = R[3 * Nn + ph::2]
        assert abs(r.sum()) <= 1e-12 * np.abs(r).sum()
