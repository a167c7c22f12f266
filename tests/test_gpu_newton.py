"""The nonlinear step on the GPU (residual of Appendix B.1, Newton with backtracking line search,
per-Newton Jacobian re-assembly on the device and flow refresh) against its CPU reference (oracle/newton.py on
residual.c, synth's CPU Jacobian and the oracle's FGMRES):
  * tsp_residual / tsp_masses equal the oracle's to rounding at displaced, perturbed states;
  * one and two implicit time steps (BHP ramp): the same number of Newton iterations, the same residual history to
    the linear solves' tolerance, the same final state; the Newton residual falls by >= 1e-6."""
import numpy as np
import pytest

import oracle
import synth
from oracle.newton import newton_step as oracle_newton_step

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def _setup(cfg, **kw):
    f = synth.fields(cfg, x_rand=False, **kw)
    prm = dict(f["params"])
    s = synth.sizes(prm["nx"], prm["ny"], prm["nz"])
    Nn = s["Nn"]
    x0 = np.zeros(s["n"])
    x0[3 * Nn::2] = f["sat"]
    x0[3 * Nn + 1::2] = f["pres"]
    ref_o = dict(E=f["E"], perm=f["perm"], phi0=f["phi"], pref=f["pres"], well=f["well"])
    ref_g = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in
             dict(E=f["E"], perm=f["perm"], phi=f["phi"], pres=f["pres"], well=f["well"]).items()}
    return prm, f, s, x0, ref_o, ref_g


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("cfg,kw", [("C1", dict(state_dp=1e6)), ("ST0", dict(nx=12, ny=12, nz=8)),
                                    ("S10", dict(nx=6, ny=8, nz=14, burden=3))])
def test_residual_and_masses_equal_the_oracle(dev, cfg, kw):
    from paper_1812_05540_b200 import masses, residual
    prm, f, s, x0, ref_o, ref_g = _setup(cfg, **kw)
    Nn, Nc = s["Nn"], s["Nc"]
    rng = np.random.default_rng(4)
    x = x0.copy()
    nbot = (prm["nx"] + 1) * (prm["ny"] + 1)
    x[3 * nbot:3 * Nn] = 1e-3 * rng.uniform(-1, 1, 3 * (Nn - nbot))
    x[3 * Nn::2] = np.clip(x[3 * Nn::2] + 0.05 * rng.uniform(-1, 1, Nc), 0, 1)
    x[3 * Nn + 1::2] += 1e5 * rng.uniform(-1, 1, Nc)
    mprev = oracle.masses(prm, ref_o, x0)
    mg = masses(prm, ref_g, _cuda(x0))
    np.testing.assert_allclose(mg.cpu().numpy(), mprev, rtol=1e-13)
    ro = oracle.residual(prm, ref_o, x, mprev, prm["dt"])
    rg = residual(prm, ref_g, _cuda(x), _cuda(mprev), prm["dt"]).cpu().numpy()
    for sl in (slice(0, 3 * Nn), slice(3 * Nn, None, 2), slice(3 * Nn + 1, None, 2)):
        assert np.linalg.norm(rg[sl] - ro[sl]) <= 1e-11 * np.linalg.norm(ro[sl])


def _run(cfg, kw, nsteps, dev, ramp=2):
    from paper_1812_05540_b200 import Tsp, assemble, masses, residual
    prm, f, s, x0, ref_o, ref_g = _setup(cfg, **kw)
    Nn = s["Nn"]
    dbhp = prm["well_dbhp"]
    # initial-state momentum equilibrium (u measures the displacement since t0)
    m0 = oracle.masses(prm, ref_o, x0)
    roff_o = oracle.residual(prm, ref_o, x0, m0, prm["dt"])[:3 * Nn]
    roff_g = residual(prm, ref_g, _cuda(x0), _cuda(m0), prm["dt"])[:3 * Nn].contiguous()
    # the handle: the Jacobian at x0 assembled on the device
    ap = assemble(prm, dict(f, phi0=f["phi"]))
    g = Tsp(ap)
    g.setup(1)                                                # TSP_SETUP_MECH: once per simulation
    xo, xg = x0.copy(), _cuda(x0)
    out = []
    for step in range(nsteps):
        p_step = dict(prm, well_dbhp=dbhp * min(1.0, (step + 1) / ramp))   # BHP ramp
        mo = oracle.masses(p_step, ref_o, xo)
        mg = masses(p_step, ref_g, xg)
        io = oracle_newton_step(p_step, ref_o, xo, mo, prm["dt"], r_off=roff_o)
        ig = g.newton_step(p_step, ref_g, xg, mg, prm["dt"], r_off=roff_g)
        out.append((io, ig, xo.copy(), xg.cpu().numpy()))
    g.close()
    return out, s


@pytest.mark.parametrize("cfg,kw,nsteps", [("C1", {}, 2), (None, dict(nx=10, ny=9, nz=20, recipe=2, perm_sigma=2.0), 2),
                                           ("ST0", dict(nx=12, ny=12, nz=8), 1)])
def test_newton_steps_match_the_oracle(dev, cfg, kw, nsteps):
    out, s = _run(cfg, kw, nsteps, dev)
    Nn = s["Nn"]
    for step, (io, ig, xo, xg) in enumerate(out):
        assert io["status"] == "OK" and ig["status"] == "OK", (step, io, ig)
        assert io["newton_iters"] == ig["newton_iters"], (step, io["res_hist"], ig["res_hist"])
        assert ig["res_hist"][-1] <= 1e-6 * ig["res_hist"][0]
        # residual histories agree to the linear tolerance (same Jacobians, FGMRES to 1e-8 on both sides)
        for a, b in zip(io["res_hist"], ig["res_hist"]):
            assert abs(a - b) <= 1e-5 * io["res_hist"][0], (step, io["res_hist"], ig["res_hist"])
        for sl in (slice(0, 3 * Nn), slice(3 * Nn, None, 2), slice(3 * Nn + 1, None, 2)):
            assert np.linalg.norm(xg[sl] - xo[sl]) <= 1e-6 * max(np.linalg.norm(xo[sl]), 1e-30), (step, sl)


def test_newton_step_is_rank_invariant(dev):
    """Two z-slab ranks on the in-process communicator, each with its slab's handle (device assembly from the global
    fields): one Newton time step gives BITWISE the one-rank state, residual history and iteration counts (the state
    and the residual are gathered, the norms taken over the gathered residual, the linear solves are P-invariant)."""
    import threading
    from paper_1812_05540_b200 import LocalWorld, Tsp, TSP_COMM_LOCAL, assemble
    kw = dict(nx=12, ny=10, nz=64, recipe=2, perm_sigma=2.0)
    prm, f, s, x0, ref_o, ref_g = _setup(None, **kw)
    Nn = s["Nn"]
    m0 = oracle.masses(prm, ref_o, x0)
    roff = oracle.residual(prm, ref_o, x0, m0, prm["dt"])[:3 * Nn]

    def run(P):
        world = LocalWorld(P) if P > 1 else None
        maxima, lock, barrier = [None] * P, threading.Lock(), threading.Barrier(P)
        out, errs = [None] * P, []

        def gmax(r):
            def fn(m):
                with lock:
                    maxima[r] = m
                barrier.wait()
                return list(np.max(np.array(maxima), axis=0))
            return fn

        def body(r):
            try:
                st = torch.cuda.Stream()
                with torch.cuda.stream(st):
                    _, _, n0, nn, c0, ncl = synth.slab_partition(prm["nx"], prm["ny"], prm["nz"], 16, r, P)
                    ap = assemble(prm, dict(f, phi0=f["phi"]), rank=r, nranks=P, stream=st, global_max=gmax(r))
                    kwc = dict(rank=r, nranks=P, comm_kind=TSP_COMM_LOCAL, comm_arg=world.h) if P > 1 else {}
                    g = Tsp(ap, stream=st, **kwc)
                    g.setup(1)
                    xl = np.concatenate([x0[3 * n0:3 * (n0 + nn)], x0[3 * Nn + 2 * c0:3 * Nn + 2 * (c0 + ncl)]])
                    x = _cuda(xl)
                    info = g.newton_step(prm, ref_g, x, None, prm["dt"], r_off=_cuda(roff[3 * n0:3 * (n0 + nn)]))
                    torch.cuda.synchronize()
                    out[r] = (x.cpu().numpy(), info, nn)
                    g.close()
            except Exception as e:   # pragma: no cover - surfaced below
                errs.append(e)

        ts = [threading.Thread(target=body, args=(r,)) for r in range(P)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        if world:
            world.close()
        if errs:
            raise errs[0]
        return out

    (x1, i1, _), = run(1)
    parts = run(2)
    u = np.concatenate([p[0][:3 * p[2]] for p in parts])
    fl = np.concatenate([p[0][3 * p[2]:] for p in parts])
    assert i1["status"] == "OK"
    assert np.array_equal(np.concatenate([u, fl]), x1)
    for p in parts:
        assert p[1]["res_hist"] == i1["res_hist"] and p[1]["lin_hist"] == i1["lin_hist"]
