"""GPU parity of the setup variants and of the second-stage options
(NEXT-f2: hybrid block Gauss-Seidel, repeated sweeps) against the oracle: true-IMPES
(eq:CPR_CSL), diagonal A_ps in step 4, fixed-stress modulus scale (remark
P:443) and RSL fixed stress (eq:FS_RSL).  Same bars as tests/test_gpu_parity.py:
D^(CPR) and the pressure hierarchy bit-exact, apply <= 1e-10, FGMRES +-1.  RSL goes
through V-cycles (rounding differs), so its D_fs is compared to 1e-10 and the rest
by the solve.  Plus P-invariance of the sharded true-IMPES / RSL (z-slabs, in-process
communicator)."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

VARIANTS = {
    "true": dict(cpr_mode=1),
    "diag_aps": dict(aps_mode=1),
    "true_diag": dict(cpr_mode=1, aps_mode=1),
    "scale": dict(fs_modulus_scale=2.0),
    "rsl": dict(fs_mode=1, rsl_iters=2),
    # NEXT-f2: the second stage
    "bgs3": dict(second_stage=1, local_sweeps=3),
    "ilu2": dict(local_sweeps=2),
}
PROBLEMS = {
    "C1": dict(config="C1"),
    "R1": dict(nx=19, ny=7, nz=21, recipe=2, perm_sigma=2.0),
}


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def _gen(name):
    kw = dict(PROBLEMS[name])
    cfg = kw.pop("config", None)
    return synth.generate(cfg, **kw)


_cache = {}


def _pair(pname, vname):
    key = (pname, vname)
    if key not in _cache:
        from paper_1812_05540_b200 import Tsp
        pb = _gen(pname)
        o = oracle.Oracle(pb, **VARIANTS[vname]).setup()
        g = Tsp(pb, **VARIANTS[vname]).setup()
        _cache.clear()
        _cache[key] = (pb, o, g)
    return _cache[key]


def _cuda(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("pname", list(PROBLEMS))
@pytest.mark.parametrize("vname", list(VARIANTS))
def test_variant_parity(dev, pname, vname):
    pb, o, g = _pair(pname, vname)
    dss_o, dps_o, fs_o = o.cpr()
    dss_g, dps_g, fs_g = g.cpr()
    if vname == "rsl":
        assert np.abs(fs_g - fs_o).max() <= 1e-10 * np.abs(fs_o).max()
    else:
        assert np.array_equal(fs_g, fs_o)
        assert np.array_equal(dss_g, dss_o) and np.array_equal(dps_g, dps_o)
        H_o, H_g = o.hierarchy(1), g.hierarchy(1)
        assert len(H_o) == len(H_g)
        for lo, lg in zip(H_o, H_g):
            for k in ("A_rp", "A_ci", "A_v", "dl1"):
                assert np.array_equal(lo[k], lg[k]), k
            if not lo["coarsest"]:
                for k in ("agg", "P_rp", "P_ci", "P_v"):
                    assert np.array_equal(lo[k], lg[k]), k
        v = np.random.default_rng(12).uniform(-1, 1, pb.n)
        z = torch.empty(pb.n, dtype=torch.float64, device=dev)
        g.apply_preconditioner(_cuda(v), z)
        torch.cuda.synchronize()
        ref = o.apply(v)
        assert np.linalg.norm(z.cpu().numpy() - ref) <= 1e-10 * np.linalg.norm(ref)
    xo, io = o.solve(pb.b, rtol=1e-8, m=64)
    x = torch.zeros(pb.n, dtype=torch.float64, device=dev)
    ig = g.solve(_cuda(pb.b), x, rtol=1e-8, restart=64)
    assert ig["status"] == "OK" and io["status"] == 0
    assert abs(ig["iterations"] - io["iterations"]) <= 1
    assert ig["true_relres"] <= 1e-8


def test_rsl_needs_mechanics_first(dev):
    from paper_1812_05540_b200 import Tsp, TSP_SETUP_FLOW
    pb = _gen("C1")
    g = Tsp(pb, fs_mode=1)
    with pytest.raises(RuntimeError):
        g.setup(TSP_SETUP_FLOW)


@pytest.mark.parametrize("vname", ["true", "rsl", "bgs3"])
def test_variant_sharded_bitwise(dev, vname):
    """z-slabs (P = 2, 4): D^(CPR), D_fs, one apply and the FGMRES solution bitwise equal to P = 1
    (true-IMPES needs the column entries of the neighbour ranks' boundary rows)."""
    from test_gpu_multirank import _run_ranks, _glue
    pb = synth.generate(nx=12, ny=10, nz=64, recipe=2, perm_sigma=2.0)
    v_glob = np.random.default_rng(21).uniform(-1, 1, pb.n)

    def work(r, g, lp):
        g.setup()
        loc = g.n != pb.n
        v = lp.local(v_glob, pb.Nn) if loc else v_glob
        b = lp.local(pb.b, pb.Nn) if loc else pb.b
        g.nc_local = lp.Nc if loc else pb.Nc
        dss, dps, fs = g.cpr()
        z = torch.empty(len(v), dtype=torch.float64, device="cuda")
        g.apply_preconditioner(torch.from_numpy(np.ascontiguousarray(v)).cuda(), z)
        x = torch.zeros_like(z)
        info = g.solve(torch.from_numpy(np.ascontiguousarray(b)).cuda(), x)
        torch.cuda.synchronize()
        return dict(z=z.cpu().numpy(), x=x.cpu().numpy(), dss=dss, dps=dps, fs=fs, info=info)

    one = _run_ranks(pb, 1, work, **VARIANTS[vname])[0]
    for P in (2, 4):
        many = _run_ranks(pb, P, work, **VARIANTS[vname])
        parts = list(zip(many, [synth.local_problem(pb, r, P) for r in range(P)]))
        for key in ("z", "x"):
            assert np.array_equal(_glue(parts, key, pb, P), one[key]), (P, key)
        for key in ("dss", "dps", "fs"):
            assert np.array_equal(np.concatenate([m[key] for m in many]), one[key]), (P, key)
        assert {m["info"]["iterations"] for m in many} == {one["info"]["iterations"]}
