"""TEST INFRASTRUCTURE ONLY: the CPU reference of the nonlinear step, the same algorithm as
tsp_newton_step on the oracle's pieces -- the residual of Appendix B.1 (residual.c, pinned by
tests/test_oracle_newton.py), the CPU Jacobian at the state (synth.assemble_state, pinned by tests/test_synth.py
and by the finite-difference test) and the oracle's two-stage FGMRES (oracle.c).

Per Newton iteration: the Jacobian at x (porosity with the strain, s, p) and its row scales S_k (the step's first
ones, S0, measure the residual); converged when ||S0 r|| <= rtol ||S0 r_0||; J y = -S_k r by FGMRES(64) to lin_rtol;
dx = (y_u, y_s, p_unit y_p); x += alpha dx with alpha halved (at most max_halvings times) until
||S0 r(x + alpha dx)|| <= (1 - 1e-4 alpha) ||S0 r(x)||; saturations clipped to [0, 1]."""
import numpy as np

from . import Oracle, porosity, residual


def _wnorm(r, nu, S):
    w = np.empty_like(r)
    w[:nu] = S[0]
    w[nu::2] = S[1]
    w[nu + 1::2] = S[2]
    return float(np.sqrt(np.sum((w * r) ** 2)))


def newton_step(params, ref, x, mprev, dt, r_off=None, rtol=1e-6, atol=0.0, max_newton=12, lin_rtol=1e-8,
                max_halvings=5, **oracle_opts):
    """One implicit time step; x (numpy, [u | (s, p [Pa])]) is updated in place.  ref: E, perm, phi0, pref, well."""
    import synth
    params = dict(params, dt=dt)                      # the Jacobian of this step's time step
    nx, ny, nz = params["nx"], params["ny"], params["nz"]
    nu = 3 * (nx + 1) * (ny + 1) * (nz + 1)
    info = dict(newton_iters=0, lin_iters=0, halvings=0, res_hist=[], lin_hist=[], status="NOT_CONVERGED")
    S0, norm0 = None, 0.0

    def rc_of(xx):
        r = residual(params, ref, xx, mprev, dt)
        if r_off is not None:
            r[:nu] -= r_off
        return r

    for it in range(1000):
        phi = porosity(params, ref, x)
        J = synth.assemble_state(params, ref["E"], ref["perm"], phi, x[nu::2], x[nu + 1::2], phi0=ref["phi0"])
        S = J.scales.copy()
        if it == 0:
            S0 = S
        r = rc_of(x)
        nrm = _wnorm(r, nu, S0)
        if it == 0:
            norm0 = nrm
            info["res0"] = nrm
        info["res"] = nrm
        info["res_hist"].append(nrm)
        if nrm <= atol or nrm <= rtol * norm0 or norm0 == 0.0:
            info["status"] = "OK"
            break
        if it >= max_newton:
            break
        w = np.empty_like(r)
        w[:nu] = S[0]
        w[nu::2] = S[1]
        w[nu + 1::2] = S[2]
        o = Oracle(J, **oracle_opts).setup()
        y, li = o.solve(-w * r, rtol=lin_rtol, m=64)
        info["lin_iters"] += li["iterations"]
        info["lin_hist"].append(li["iterations"])
        d = y.copy()
        d[nu + 1::2] *= params["p_unit"]
        alpha, hv = 1.0, 0
        while True:
            xt = x + alpha * d
            xt[nu::2] = np.clip(xt[nu::2], 0.0, 1.0)
            nt = _wnorm(rc_of(xt), nu, S0)
            if nt <= (1.0 - 1e-4 * alpha) * nrm or hv >= max_halvings:
                break
            alpha *= 0.5
            hv += 1
            info["halvings"] += 1
        x[:] = xt
        info["newton_iters"] = it + 1
    return info
