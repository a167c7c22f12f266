"""GPU parity of the value-only flow refresh (DESIGN.md R-refresh; the oracle's version is
pinned in tests/test_oracle_refresh.py): tsp_update_values (a Newton step's new values on the same patterns,
P:519) followed by tsp_setup(FLOW | REFRESH) keeps the pressure AMG's strength flags, aggregates and
patterns and recomputes every value.  Compared with the oracle's update_values + setup_flow(refresh): pressure
hierarchy bit-exact, D_ss / D_ps / D_fs bit-exact, operator <= 1e-13, one Algorithm 1 application <= 1e-10,
FGMRES +-1."""
import threading

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def _cuda(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _same_hier(Ha, Hb, values=True):
    assert len(Ha) == len(Hb)
    for lvl, (la, lb) in enumerate(zip(Ha, Hb)):
        keys = ("A_rp", "A_ci") + (("A_v", "dl1") if values else ())
        if not la["coarsest"]:
            keys += ("agg", "P_rp", "P_ci") + (("P_v",) if values else ())
        for k in keys:
            assert np.array_equal(la[k], lb[k]), (lvl, k)


def _apply(g, v, dev):
    z = torch.empty(len(v), dtype=torch.float64, device=dev)
    g.apply_preconditioner(_cuda(v), z)
    torch.cuda.synchronize()
    return z.cpu().numpy()


@pytest.mark.parametrize("smoother", [0, 1])
def test_refresh_with_unchanged_values_is_the_full_setup(dev, smoother):
    """Same values: the GPU refresh reproduces the GPU's own full flow setup bit for bit (pressure hierarchy and
    one application), and both equal the oracle's refresh."""
    from paper_1812_05540_b200 import Tsp
    pb = synth.generate(nx=10, ny=9, nz=20, recipe=2, perm_sigma=2.0)
    full = Tsp(pb, amg_smoother=smoother).setup()
    g = Tsp(pb, amg_smoother=smoother).setup()
    g.update_values(pb).setup_flow(refresh=True)
    _same_hier(full.hierarchy(1), g.hierarchy(1))
    v = np.random.default_rng(3).uniform(-1, 1, pb.n)
    assert np.array_equal(_apply(full, v, dev), _apply(g, v, dev))
    o = oracle.Oracle(pb, amg_smoother=smoother).setup()
    o.update_values(pb).setup_flow(refresh=True)
    _same_hier(o.hierarchy(1), g.hierarchy(1))
    full.close(); g.close()


@pytest.mark.parametrize("name,kw", [("C2", dict(config="C2")),
                                     ("R1", dict(nx=19, ny=7, nz=21, recipe=2, perm_sigma=2.0))])
def test_newton_step_refresh_parity(dev, name, kw):
    """A changed linearisation state (hydrostatic + 2 MPa, R-state), same grid: the GPU after update_values +
    refresh equals the oracle after the same calls -- pressure hierarchy (old aggregates, new values) and the
    CPR / fixed-stress diagonals bit-exact, operator <= 1e-13, applications <= 1e-10, FGMRES +-1."""
    from paper_1812_05540_b200 import Tsp
    kw = dict(kw)
    cfg = kw.pop("config", None)
    pb1 = synth.generate(cfg, **kw)
    pb2 = synth.generate(cfg, state_dp=2e6, **kw)
    assert not np.array_equal(pb1.ff_val, pb2.ff_val)
    g = Tsp(pb1).setup()
    H1 = g.hierarchy(1)
    g.update_values(pb2)
    o = oracle.Oracle(pb1).setup()
    o.update_values(pb2)
    # the operator switches at once; the preconditioner waits for the flow phase on the new values
    x = np.random.default_rng(5).uniform(-1, 1, pb2.n)
    y = torch.empty(pb2.n, dtype=torch.float64, device=dev)
    g.apply_operator(_cuda(x), y)
    torch.cuda.synchronize()
    ref = o.operator(x)
    assert np.linalg.norm(y.cpu().numpy() - ref) <= 1e-13 * np.linalg.norm(ref)
    from paper_1812_05540_b200 import TspError
    with pytest.raises(TspError, match="STATE"):
        _apply(g, x, dev)
    g.setup_flow(refresh=True)
    o.setup_flow(refresh=True)
    H2 = g.hierarchy(1)
    _same_hier(H1, H2, values=False)                      # frozen aggregation: same structure
    _same_hier(o.hierarchy(1), H2)                        # and the oracle's values, bit for bit
    for a, b in zip(o.cpr(), g.cpr()):
        assert np.array_equal(a, b)
    for seed in (7, 8):
        v = np.random.default_rng(seed).uniform(-1, 1, pb2.n)
        ref = o.apply(v)
        assert np.linalg.norm(_apply(g, v, dev) - ref) <= 1e-10 * np.linalg.norm(ref)
    xg = torch.zeros(pb2.n, dtype=torch.float64, device=dev)
    ig = g.solve(_cuda(pb2.b), xg, rtol=1e-8)
    _, io = o.solve(pb2.b, rtol=1e-8)
    assert ig["status"] == "OK" and io["status"] == 0 and abs(ig["iterations"] - io["iterations"]) <= 1, (ig, io)
    assert ig["true_relres"] <= 1e-8
    g.close()


def test_update_then_mech_setup_equals_a_fresh_handle(dev):
    """update_values + tsp_setup(MECH | FLOW) = tsp_create on the new values + setup, bitwise (both hierarchies,
    the structured A_uu / level-0 SDC copies rebuilt from the new A_uu, one application, the operator)."""
    from paper_1812_05540_b200 import Tsp
    pb1 = synth.generate(nx=11, ny=9, nz=18, recipe=2, perm_sigma=2.0)
    pb2 = synth.generate(nx=11, ny=9, nz=18, recipe=2, perm_sigma=2.0, state_dp=3e6)
    pb2.uu_val = pb2.uu_val * 1.5                          # a different mechanics block too
    g = Tsp(pb1).setup()
    g.update_values(pb2).setup()
    f = Tsp(pb2).setup()
    for w in (0, 1):
        _same_hier(f.hierarchy(w), g.hierarchy(w))
    v = np.random.default_rng(9).uniform(-1, 1, pb2.n)
    assert np.array_equal(_apply(f, v, dev), _apply(g, v, dev))
    yf, yg = (torch.empty(pb2.n, dtype=torch.float64, device=dev) for _ in range(2))
    f.apply_operator(_cuda(v), yf)
    g.apply_operator(_cuda(v), yg)
    torch.cuda.synchronize()
    assert torch.equal(yf, yg)
    f.close(); g.close()


def test_asymmetric_update_falls_back_to_the_generic_layout(dev):
    """New A_uu values that break the symmetry the structured layout assumes: the operator moves to the generic
    SELL copy and still equals the oracle's operator on the new values."""
    from paper_1812_05540_b200 import Tsp
    pb1 = synth.generate("C1")
    pb2 = synth.generate("C1")
    pb2.uu_val = pb2.uu_val.copy()
    q = pb2.uu_rowptr[400] + 1
    pb2.uu_val[q, 0, 1] += 0.25 * abs(pb2.uu_val[q, 0, 1]) + 1e-3   # (x,y) entry: symmetric in the original
    g = Tsp(pb1).setup()
    g.update_values(pb2)
    o = oracle.Oracle(pb1).setup()
    o.update_values(pb2)
    x = np.random.default_rng(2).uniform(-1, 1, pb2.n)
    y = torch.empty(pb2.n, dtype=torch.float64, device=dev)
    g.apply_operator(_cuda(x), y)
    torch.cuda.synchronize()
    ref = o.operator(x)
    assert np.linalg.norm(y.cpu().numpy() - ref) <= 1e-13 * np.linalg.norm(ref)
    g.close()


def test_update_with_a_new_pattern_is_refused_and_harmless(dev):
    from paper_1812_05540_b200 import Tsp, TspError
    pb = synth.generate("C1")
    g = Tsp(pb).setup()
    v = np.random.default_rng(1).uniform(-1, 1, pb.n)
    z0 = _apply(g, v, dev)
    pb2 = synth.generate("C1")
    pb2.ff_col = pb2.ff_col.copy()
    pb2.ff_col[1], pb2.ff_col[2] = pb2.ff_col[2], pb2.ff_col[1]
    with pytest.raises(TspError):
        g.update_values(pb2)
    pb3 = synth.generate("C1")
    pb3.fs = -pb3.fs
    with pytest.raises(TspError):
        g.update_values(pb3)
    assert np.array_equal(z0, _apply(g, v, dev))          # refused updates leave the handle as it was
    with pytest.raises(TspError):                         # REFRESH without FLOW
        g.setup(4)
    g.close()
    g = Tsp(pb)
    with pytest.raises(TspError):                         # refresh before any flow setup
        g.setup_flow(refresh=True)
    g.close()


def test_refresh_is_rank_invariant(dev):
    """P = 2 ranks (in-process communicator): update_values + refresh gives BITWISE the P = 1 pressure hierarchy
    and application (distributed levels, ghost P rows and gathered coarse levels rebuilt with frozen aggregates)."""
    from paper_1812_05540_b200 import LocalWorld, Tsp, TSP_COMM_LOCAL
    grid = dict(nx=12, ny=10, nz=64, recipe=2, perm_sigma=2.0)
    pb1 = synth.generate(**grid)
    pb2 = synth.generate(state_dp=2e6, **grid)
    v_glob = np.random.default_rng(11).uniform(-1, 1, pb1.n)

    def run(P):
        world = LocalWorld(P) if P > 1 else None
        out, errs = [None] * P, []

        def body(r):
            try:
                s = torch.cuda.Stream()
                with torch.cuda.stream(s):
                    if P == 1:
                        g, lp2, v = Tsp(pb1, stream=s), pb2, v_glob
                    else:
                        lp1, lp2 = synth.local_problem(pb1, r, P), synth.local_problem(pb2, r, P)
                        g = Tsp(lp1, stream=s, rank=r, nranks=P, comm_kind=TSP_COMM_LOCAL, comm_arg=world.h,
                                replicate_rows=200)
                        v = lp1.local(v_glob, pb1.Nn)
                    g.setup()
                    g.update_values(lp2).setup_flow(refresh=True)
                    dv = _cuda(v)
                    z = torch.empty_like(dv)
                    g.apply_preconditioner(dv, z)
                    torch.cuda.synchronize()
                    H = [g.level(1, l) for l in range(g.num_levels(1))]
                    out[r] = (z.cpu().numpy(), H, [g.level_dist(1, l) for l in range(g.num_levels(1))])
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

    (z1, H1, _), = run(1)
    parts = run(2)
    lps = [synth.local_problem(pb1, r, 2) for r in range(2)]
    u = np.concatenate([p[0][:3 * lp.Nn] for p, lp in zip(parts, lps)])
    f = np.concatenate([p[0][3 * lp.Nn:] for p, lp in zip(parts, lps)])
    assert np.array_equal(np.concatenate([u, f]), z1)
    assert any(d["dist"] for d in parts[0][2])              # some refreshed level was distributed
    for lvl, (l1,) in enumerate(zip(H1)):
        dist = parts[0][2][lvl]["dist"]
        if dist:
            A_v = np.concatenate([p[1][lvl]["A_v"] for p in parts])
        else:
            A_v = parts[0][1][lvl]["A_v"]
        assert np.array_equal(l1["A_v"], A_v), lvl
