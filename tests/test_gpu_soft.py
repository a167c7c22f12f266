"""Soft-error semantics through the C-ABI against the oracle (include/tsp.h
tsp_stats counters): the inputs of tests/test_oracle_soft.py (where the oracle's behaviour is pinned) run on
the CUDA path; counters equal, hierarchies bit-exact, one application <= 1e-10, FGMRES +-1."""
import numpy as np
import pytest

import oracle
from test_oracle_soft import singular_pivot_problem, stagnating_problem, zero_dss_problem

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def _cuda(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _compare(pb, opts, dev, apply_tol=1e-10, solve=True):
    from paper_1812_05540_b200 import Tsp
    o = oracle.Oracle(pb, **opts).setup()
    g = Tsp(pb, **opts).setup()
    st, co = g.stats(), o.counters()
    assert (st["skipped_dss"], st["perturbed_pivots"], st["coarsening_fallbacks"]) == \
        (co["skipped_dss"], co["perturbed"], co["fallbacks"])
    for which in (0, 1):
        H_o, H_g = o.hierarchy(which), g.hierarchy(which)
        assert len(H_o) == len(H_g)
        for lo, lg in zip(H_o, H_g):
            for k in ("A_rp", "A_ci", "A_v", "dl1") + (() if lo["coarsest"] else ("agg", "P_rp", "P_ci", "P_v")):
                assert np.array_equal(lo[k], lg[k]), (which, k)
    z = torch.empty(pb.n, dtype=torch.float64, device=dev)
    for seed in (1, 2):
        v = np.random.default_rng(seed).uniform(-1, 1, pb.n)
        g.apply_preconditioner(_cuda(v), z)
        torch.cuda.synchronize()
        ref = o.apply(v)
        assert np.linalg.norm(z.cpu().numpy() - ref) <= apply_tol * np.linalg.norm(ref)
    if solve:
        xo, io = o.solve(pb.b, rtol=1e-8, m=64)
        x = torch.zeros(pb.n, dtype=torch.float64, device=dev)
        ig = g.solve(_cuda(pb.b), x, rtol=1e-8)
        assert ig["status"] == "OK" and io["status"] == 0 and abs(ig["iterations"] - io["iterations"]) <= 1
    g.close()
    return st


def test_zero_dss_row(dev):
    """a zero D_ss row is skipped (z_s = 0, S_pp row uncorrected) and counted, on both sides."""
    pb, _ = zero_dss_problem(4)
    st = _compare(pb, {}, dev)
    assert st["skipped_dss"] == 1


def test_zero_dss_row_larger(dev):
    """The same on a grid with several ILU tiles and z-blocks, three zeroed rows."""
    pb, _ = zero_dss_problem(0, nx=19, ny=7, nz=21, recipe=2, perm_sigma=2.0)
    for cell in (1000, 2792):
        q = pb.ff_rowptr[cell] + int(np.flatnonzero(pb.ff_col[pb.ff_rowptr[cell]:pb.ff_rowptr[cell + 1]] == cell)[0])
        pb.ff_val[q, 0, 0] = 0.0
    st = _compare(pb, {}, dev)
    assert st["skipped_dss"] == 3


def test_singular_ilu_pivot(dev):
    """a singular tile pivot is perturbed by 1e-12 max|U_KK| and counted, on both sides.  The perturbed
    pivot has cond ~ 1e12, so rounding differences between the GPU's DILU form and the oracle's IKJ
    factorisation (same operator, different association) are amplified up to cond * eps ~ 1e-4 (measured
    4.8e-7 on the B200); the bar is 1e-5 for this degenerate case only."""
    pb, _ = singular_pivot_problem(0)
    st = _compare(pb, {}, dev, apply_tol=1e-5, solve=False)
    assert st["perturbed_pivots"] == 1


def test_coarsening_stagnation(dev):
    """a level without aggregates stops both hierarchies with a dense solve, counted, bit-exact."""
    pb, kw = stagnating_problem()
    st = _compare(pb, kw, dev)
    assert st["coarsening_fallbacks"] == 2


def test_stagnation_beyond_dense_limit_is_an_error(dev):
    """D4: a stagnated level above 4096 rows is TSP_ERR_SINGULAR (-7) on the GPU and a setup failure in the
    oracle."""
    import synth
    from paper_1812_05540_b200 import Tsp, TspError
    pb = synth.generate(nx=1, ny=1, nz=4200, recipe=1)
    with pytest.raises(RuntimeError):
        oracle.Oracle(pb, zblock=1).setup()
    g = Tsp(pb, zblock=1)
    with pytest.raises(TspError) as e:
        g.setup()
    assert e.value.status == -7
    g.close()
