"""GPU parity of the Chebyshev AMG smoother (tsp_options.amg_smoother = 2; north_star "fused Jacobi/Chebyshev or
l1-Jacobi AMG smoothers"; DESIGN.md R-cheb; the oracle's version is pinned in tests/test_oracle_cheb.py): one
Algorithm 1 application <= 1e-10 against the oracle, FGMRES +-1, and -- unlike Gauss-Seidel -- the z-slab
decomposition: P = 2 ranks bitwise equal to P = 1."""
import threading

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

PROBLEMS = {
    "C1": (dict(config="C1"), {}),
    "C1-deg3": (dict(config="C1"), dict(amg_cheb_degree=3, amg_cheb_lower=0.1)),
    "C2": (dict(config="C2"), {}),
    "R1": (dict(nx=19, ny=7, nz=21, recipe=2, perm_sigma=2.0), {}),
    "ST1": (dict(config="ST1"), {}),
    "C2-pressure-only": (dict(config="C2"), dict(amg_smoother=0, amg_smoother_p=2)),
    "R1-mech-only": (dict(nx=19, ny=7, nz=21, recipe=2, perm_sigma=2.0), dict(amg_smoother_p=0)),
}


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def _cuda(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("name", list(PROBLEMS))
def test_cheb_parity(dev, name):
    from paper_1812_05540_b200 import Tsp
    kw, extra = PROBLEMS[name]
    kw = dict(kw)
    pb = synth.generate(kw.pop("config", None), **kw)
    opts = {"amg_smoother": 2, **extra}
    o = oracle.Oracle(pb, **opts).setup()
    g = Tsp(pb, **opts).setup()
    rng = np.random.default_rng(5)
    z = torch.empty(pb.n, dtype=torch.float64, device=dev)
    nu = 3 * pb.Nn
    for v in (pb.b, rng.uniform(-1, 1, pb.n)):
        g.apply_preconditioner(_cuda(v), z)
        torch.cuda.synchronize()
        ref = o.apply(v)
        got = z.cpu().numpy()
        assert np.linalg.norm(got - ref) <= 1e-10 * np.linalg.norm(ref)
        assert np.linalg.norm(got[:nu] - ref[:nu]) <= 1e-10 * np.linalg.norm(ref[:nu])
    x = torch.zeros(pb.n, dtype=torch.float64, device=dev)
    ig = g.solve(_cuda(pb.b), x, rtol=1e-8)
    _, io = o.solve(pb.b, rtol=1e-8)
    assert ig["status"] == "OK" and io["status"] == 0 and abs(ig["iterations"] - io["iterations"]) <= 1, (ig, io)
    g.close()


def test_cheb_is_rank_invariant(dev):
    from paper_1812_05540_b200 import LocalWorld, Tsp, TSP_COMM_LOCAL
    pb = synth.generate(nx=12, ny=10, nz=64, recipe=2, perm_sigma=2.0)
    v_glob = np.random.default_rng(3).uniform(-1, 1, pb.n)

    def run(P):
        world = LocalWorld(P) if P > 1 else None
        out, errs = [None] * P, []

        def body(r):
            try:
                s = torch.cuda.Stream()
                with torch.cuda.stream(s):
                    if P == 1:
                        g, v, b = Tsp(pb, stream=s, amg_smoother=2), v_glob, pb.b
                    else:
                        lp = synth.local_problem(pb, r, P)
                        g = Tsp(lp, stream=s, rank=r, nranks=P, comm_kind=TSP_COMM_LOCAL, comm_arg=world.h,
                                amg_smoother=2, replicate_rows=200)
                        v, b = lp.local(v_glob, pb.Nn), lp.local(pb.b, pb.Nn)
                    g.setup()
                    dv = _cuda(v)
                    z = torch.empty_like(dv)
                    g.apply_preconditioner(dv, z)
                    x = torch.zeros_like(dv)
                    info = g.solve(_cuda(b), x, rtol=1e-8)
                    torch.cuda.synchronize()
                    out[r] = (z.cpu().numpy(), x.cpu().numpy(), info["iterations"])
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

    (z1, x1, it1), = run(1)
    parts = run(2)
    lps = [synth.local_problem(pb, r, 2) for r in range(2)]

    def glue(k):
        u = np.concatenate([p[k][:3 * lp.Nn] for p, lp in zip(parts, lps)])
        f = np.concatenate([p[k][3 * lp.Nn:] for p, lp in zip(parts, lps)])
        return np.concatenate([u, f])

    assert np.array_equal(glue(0), z1)
    assert np.array_equal(glue(1), x1)
    assert parts[0][2] == parts[1][2] == it1
