"""GPU parity of the paper's Gauss-Seidel AMG smoother (tsp_options.amg_smoother = 1; DESIGN.md R-gs;
the oracle's version is pinned in tests/test_oracle_gs.py): colourings identical to the oracle's on every level,
hierarchies bit-exact (the smoother does not touch the setup arithmetic), one Algorithm 1 application <= 1e-10,
FGMRES +-1 with fewer iterations than l1-Jacobi."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

PROBLEMS = {
    "C1": dict(config="C1"),
    "C2": dict(config="C2"),
    "R1": dict(nx=19, ny=7, nz=21, recipe=2, perm_sigma=2.0),
    "ST1": dict(config="ST1"),
}


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def _cuda(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("name", list(PROBLEMS))
def test_gs_parity(dev, name):
    from paper_1812_05540_b200 import Tsp
    kw = dict(PROBLEMS[name])
    pb = synth.generate(kw.pop("config", None), **kw)
    o = oracle.Oracle(pb, amg_smoother=1).setup()
    g = Tsp(pb, amg_smoother=1).setup()
    for which in (0, 1):
        H_o, H_g = o.hierarchy(which), g.hierarchy(which)
        assert len(H_o) == len(H_g)
        for lvl, (lo, lg) in enumerate(zip(H_o, H_g)):
            for k in ("A_rp", "A_ci", "A_v") + (() if lo["coarsest"] else ("agg", "P_v")):
                assert np.array_equal(lo[k], lg[k]), (which, lvl, k)
            if lo["coarsest"]:
                continue
            co, nco = o.colour(which, lvl)
            cg, blk, ncg = g.colour(which, lvl)
            assert np.array_equal(co, cg) and nco == ncg, (which, lvl)
            assert blk == (0 if lvl == 0 else 1024)
    rng = np.random.default_rng(5)
    z = torch.empty(pb.n, dtype=torch.float64, device=dev)
    nu = 3 * pb.Nn
    for v in (pb.b, rng.uniform(-1, 1, pb.n)):
        g.apply_preconditioner(_cuda(v), z)
        torch.cuda.synchronize()
        ref = o.apply(v)
        got = z.cpu().numpy()
        assert np.linalg.norm(got - ref) <= 1e-10 * np.linalg.norm(ref)
        for sl in (slice(0, nu), slice(nu, None, 2), slice(nu + 1, None, 2)):
            assert np.linalg.norm(got[sl] - ref[sl]) <= 1e-10 * np.linalg.norm(ref[sl])
    xo, io = o.solve(pb.b, rtol=1e-8)
    x = torch.zeros(pb.n, dtype=torch.float64, device=dev)
    ig = g.solve(_cuda(pb.b), x, rtol=1e-8)
    assert ig["status"] == "OK" and io["status"] == 0 and abs(ig["iterations"] - io["iterations"]) <= 1
    g2 = Tsp(pb).setup()
    x2 = torch.zeros(pb.n, dtype=torch.float64, device=dev)
    ij = g2.solve(_cuda(pb.b), x2, rtol=1e-8)
    print(f"[gs {name}] FGMRES iterations: GS {ig['iterations']} (oracle {io['iterations']}), l1-Jacobi {ij['iterations']}")
    assert ig["iterations"] <= ij["iterations"]
    g.close(); g2.close()


def test_gs_refused_on_multiple_ranks(dev):
    """R-gs is single-GPU: a sharded handle with amg_smoother = 1 is refused at setup with a message."""
    from paper_1812_05540_b200 import TspError
    from test_gpu_multirank import _run_ranks
    pb = synth.generate(nx=8, ny=8, nz=32, recipe=2, perm_sigma=1.0)
    with pytest.raises(TspError) as e:
        _run_ranks(pb, 2, lambda r, g, lp: g.setup(), amg_smoother=1)
    assert e.value.status == -1
