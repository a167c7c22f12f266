"""Row (e): z-slab decomposition.  P ranks run in ONE process on one GPU through
the library's in-process communicator (TSP_COMM_LOCAL: one host thread and one
stream per rank, device-to-device halo copies ordered by events; no kernel ever
waits on another rank).  It exercises every sharded code path except the NCCL
transport: halos of the operator, of Algorithm 1 and of the distributed AMG
levels, ghost P rows in the Galerkin product, coarse-level gathering and the
chunked deterministic reductions.  The assertion is the design invariant
(SURVEY D19-D20): results for P = 2, 4 are BITWISE identical to P = 1."""
import threading

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GRID = dict(nx=12, ny=10, nz=64, recipe=2, perm_sigma=2.0)   # 4 z-blocks of 16 planes


def _run_ranks(pb, P, work, **opts):
    """Create P handles (one thread each) on the local world, run work(rank, handle, lp)."""
    from paper_1812_05540_b200 import LocalWorld, Tsp, TSP_COMM_LOCAL
    world = LocalWorld(P)
    out, errs = [None] * P, []

    def body(r):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                lp = synth.local_problem(pb, r, P)
                if P == 1:
                    g = Tsp(pb, stream=s, **opts)
                else:
                    g = Tsp(lp, stream=s, rank=r, nranks=P, comm_kind=TSP_COMM_LOCAL, comm_arg=world.h, **opts)
                out[r] = work(r, g, lp)
                torch.cuda.synchronize()
                g.close()
        except Exception as e:   # pragma: no cover - surfaced below
            errs.append(e)

    ts = [threading.Thread(target=body, args=(r,)) for r in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    world.close()
    if errs:
        raise errs[0]
    return out


def _work(pb):
    rng = np.random.default_rng(21)
    v_glob = rng.uniform(-1, 1, pb.n)

    def work(r, g, lp):
        g.setup()
        nglob = pb.Nn
        v = lp.local(v_glob, nglob) if g.n != pb.n else v_glob
        b = lp.local(pb.b, nglob) if g.n != pb.n else pb.b
        dv = torch.from_numpy(np.ascontiguousarray(v)).cuda()
        z = torch.empty_like(dv)
        g.apply_preconditioner(dv, z)
        y = torch.empty_like(dv)
        g.apply_operator(dv, y)
        x = torch.zeros_like(dv)
        info = g.solve(torch.from_numpy(np.ascontiguousarray(b)).cuda(), x)
        torch.cuda.synchronize()
        H = {w: [(g.level_dist(w, l), g.level(w, l)) for l in range(g.num_levels(w))] for w in (0, 1)}
        return dict(z=z.cpu().numpy(), y=y.cpu().numpy(), x=x.cpu().numpy(), info=info, H=H)

    return work


def _glue(parts, key, pb, P):
    """Reassemble the global vector [u | f] from the ranks' [u_own | f_own]."""
    u = np.concatenate([p[key][:3 * lp.Nn] for p, lp in parts])
    f = np.concatenate([p[key][3 * lp.Nn:] for p, lp in parts])
    return np.concatenate([u, f])


@pytest.fixture(scope="module")
def problem():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return synth.generate(**GRID)


@pytest.mark.parametrize("P,rep", [(2, 32768), (4, 32768), (2, 64), (4, 64)])
def test_sharded_bitwise_equals_single(problem, P, rep):
    pb = problem
    one = _run_ranks(pb, 1, _work(pb), replicate_rows=rep)[0]
    many = _run_ranks(pb, P, _work(pb), replicate_rows=rep)
    parts = list(zip(many, [synth.local_problem(pb, r, P) for r in range(P)]))
    for key in ("y", "z", "x"):
        glued = _glue(parts, key, pb, P)
        assert np.array_equal(glued, one[key]), key
    its = {m["info"]["iterations"] for m in many}
    assert its == {one["info"]["iterations"]}
    assert all(m["info"]["true_relres"] == one["info"]["true_relres"] for m in many)
    # hierarchies: distributed levels glued in rank order, replicated levels identical on every rank
    for w in (0, 1):
        H1 = one["H"][w]
        assert all(len(m["H"][w]) == len(H1) for m in many)
        for l, (d1, L1) in enumerate(H1):
            dists = [m["H"][w][l][0] for m in many]
            Ls = [m["H"][w][l][1] for m in many]
            if dists[0]["dist"]:
                assert l == 0 or rep == 64
                for k in ("A_ci", "A_v", "dl1") + (() if L1["coarsest"] else ("agg", "P_v")):
                    assert np.array_equal(np.concatenate([L[k] for L in Ls]), L1[k]), (w, l, k)
                rl = np.concatenate([[0]] + [np.diff(L["A_rp"]) for L in Ls]).cumsum()
                assert np.array_equal(rl, L1["A_rp"])
            else:
                for L in Ls:
                    for k in ("A_rp", "A_ci", "A_v", "dl1"):
                        assert np.array_equal(L[k], L1[k]), (w, l, k)


def test_more_ranks_than_z_blocks_is_rejected():
    """nz = 20 has two z-blocks of 16 planes: a rank must own at least one (include/tsp.h, tsp_create), so P = 4
    is refused with TSP_ERR_INVALID_ARG and a message, on every rank, instead of hanging in a collective."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1812_05540_b200.tsp import TspError
    pb = synth.generate(nx=9, ny=7, nz=20, recipe=2, perm_sigma=1.5)
    with pytest.raises(TspError, match="more ranks than z-blocks"):
        _run_ranks(pb, 4, _work(pb))
