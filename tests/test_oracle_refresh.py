"""Pins of the oracle's value-only flow refresh (NEXT-f1; DESIGN.md R-refresh): a Newton step changes the
Jacobian's values, not its patterns (the flow setup is redone every Newton step, the mechanics
setup once).  orc_update_values + orc_setup_flow(refresh=1) keep the pressure hierarchy's strength graphs,
aggregates and patterns and recompute every value in the build's own order.  CPU only."""
import numpy as np
import pytest

import oracle
import synth


def _same_hier(Ha, Hb):
    assert len(Ha) == len(Hb)
    for la, lb in zip(Ha, Hb):
        for k in ("A_rp", "A_ci", "A_v", "dl1") + (() if la["coarsest"] else ("agg", "P_rp", "P_ci", "P_v")):
            assert np.array_equal(la[k], lb[k]), k


@pytest.mark.parametrize("smoother", [0, 1])
def test_refresh_with_unchanged_values_is_the_full_setup(smoother):
    """Same values: the frozen refresh reproduces the full flow setup bit for bit (hierarchy, D_ss, S_pp, and
    one Algorithm 1 application)."""
    pb = synth.generate(nx=10, ny=9, nz=20, recipe=2, perm_sigma=2.0)
    full = oracle.Oracle(pb, amg_smoother=smoother).setup()
    ref = oracle.Oracle(pb, amg_smoother=smoother).setup()
    ref.update_values(pb).setup_flow(refresh=True)
    _same_hier(full.hierarchy(1), ref.hierarchy(1))
    for a, b in zip(full.spp(), ref.spp()):
        assert np.array_equal(a, b)
    v = np.random.default_rng(3).uniform(-1, 1, pb.n)
    assert np.array_equal(full.apply(v), ref.apply(v))


def test_refresh_of_a_scaled_flow_block_equals_the_full_setup():
    """Flow rows scaled by 2 (A_fu, A_ff and D_fs; exact in IEEE arithmetic): strength decisions are
    scale-invariant, so the full setup keeps the same aggregates and the frozen refresh must equal it bit for
    bit; the pressure operators are exactly twice the originals."""
    pb = synth.generate(nx=10, ny=9, nz=20, recipe=2, perm_sigma=2.0)
    pb2 = synth.generate(nx=10, ny=9, nz=20, recipe=2, perm_sigma=2.0)
    pb2.ff_val = 2.0 * pb.ff_val
    pb2.fu_val = 2.0 * pb.fu_val
    pb2.fs = 2.0 * pb.fs
    o = oracle.Oracle(pb).setup()
    H1 = o.hierarchy(1)
    o.update_values(pb2).setup_flow(refresh=True)
    full2 = oracle.Oracle(pb2).setup()
    _same_hier(full2.hierarchy(1), o.hierarchy(1))
    for l1, l2 in zip(H1, o.hierarchy(1)):
        assert np.array_equal(2.0 * l1["A_v"], l2["A_v"])
    v = np.random.default_rng(4).uniform(-1, 1, pb.n)
    assert np.array_equal(full2.apply(v), o.apply(v))


def test_newton_step_refresh_keeps_the_structure_and_converges():
    """A changed linearisation state (hydrostatic pressure + 2 MPa, R-state) on the same grid: the refreshed
    hierarchy has the old aggregates and patterns and the new values, the operator is the new Jacobian, and
    FGMRES converges with the refreshed preconditioner as with a full setup (+-2 iterations)."""
    pb1 = synth.generate("C2")
    pb2 = synth.generate("C2", state_dp=2e6)
    assert not np.array_equal(pb1.ff_val, pb2.ff_val)
    o = oracle.Oracle(pb1).setup()
    H1 = o.hierarchy(1)
    o.update_values(pb2).setup_flow(refresh=True)
    H2 = o.hierarchy(1)
    for l1, l2 in zip(H1, H2):
        for k in ("A_rp", "A_ci") + (() if l1["coarsest"] else ("agg", "P_rp", "P_ci")):
            assert np.array_equal(l1[k], l2[k])
    x = np.random.default_rng(5).uniform(-1, 1, pb2.n)
    A2, _ = synth.to_scipy(pb2)
    assert np.linalg.norm(o.operator(x) - A2 @ x) <= 1e-14 * np.linalg.norm(A2 @ x)
    _, ir = o.solve(pb2.b, rtol=1e-8)
    _, ifull = oracle.Oracle(pb2).setup().solve(pb2.b, rtol=1e-8)
    assert ir["status"] == 0 and ir["true_relres"] <= 1e-8
    assert abs(ir["iterations"] - ifull["iterations"]) <= 2, (ir["iterations"], ifull["iterations"])


def test_update_with_a_new_pattern_is_refused():
    pb = synth.generate("C1")
    o = oracle.Oracle(pb).setup()
    pb2 = synth.generate("C1")
    pb2.ff_col = pb2.ff_col.copy()
    pb2.ff_col[1], pb2.ff_col[2] = pb2.ff_col[2], pb2.ff_col[1]
    with pytest.raises(ValueError):
        o.update_values(pb2)
