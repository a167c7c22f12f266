"""GPU assembly of the linearised Jacobian (tsp_assemble / tsp_assemble_scale; SURVEY NEXT-f1 "GPU assembly of the
Appendix B Jacobian") against the CPU assembler of synth/ (its oracle here; the two share no code,
only the seeded fields): patterns identical, every block value and the fixed-stress diagonals equal to rounding
(different summation order of the Gauss integrals), the row scales equal, for the BASELINE recipes, the staircase
(channel wells), the SPE10-shaped seal layers with five wells, and a z-slab split whose global row maxima come
from the ranks; and the solve on the device-assembled Jacobian takes the same FGMRES count as on the host one."""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CASES = {
    "C1": (dict(config="C1"), {}),
    "C2": (dict(config="C2"), {}),
    "C3-shape": (dict(config="C3"), dict(nx=20, ny=18, nz=24)),
    "C4-shape": (dict(config="C4"), dict(nx=24, ny=20, nz=16)),
    "ST1": (dict(config="ST1"), {}),
    "S10-shape": (dict(config="S10"), dict(nx=12, ny=22, nz=40, burden=8)),
    "R1-state": (dict(config=None), dict(nx=19, ny=7, nz=21, recipe=2, perm_sigma=2.0, state_dp=2e6)),
}


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def _host(t):
    return t.cpu().numpy()


def _compare(pb, ap, rows=None):
    """Patterns exact; values to 1e-12 of each block row's largest entry."""
    for name, bs in (("uu", 9), ("uf", 6), ("fu", 6), ("ff", 4)):
        rp, ci, v = getattr(pb, name + "_rowptr"), getattr(pb, name + "_col"), getattr(pb, name + "_val")
        if rows is not None:
            r0, nr = rows[name]
            q0, q1 = rp[r0], rp[r0 + nr]
            rp, ci, v = rp[r0:r0 + nr + 1] - q0, ci[q0:q1], v[q0:q1]
        grp, gci = _host(getattr(ap, name + "_rowptr")), _host(getattr(ap, name + "_col"))
        gv = _host(getattr(ap, name + "_val"))[:len(ci) * bs].reshape(v.shape)
        assert np.array_equal(grp, rp), name
        assert np.array_equal(gci[:len(ci)], ci), name
        scale = np.repeat(np.maximum.reduceat(np.abs(v).reshape(len(ci), -1).max(1), rp[:-1]) if len(ci) else [], np.diff(rp))
        err = np.abs(gv - v).reshape(len(ci), -1).max(1)
        assert np.all(err <= 1e-12 * np.maximum(scale, 1e-300)), (name, float((err / np.maximum(scale, 1e-300)).max()))


@pytest.mark.parametrize("name", list(CASES))
def test_gpu_assembly_equals_the_cpu_assembler(dev, name):
    from paper_1812_05540_b200 import assemble
    base, over = CASES[name]
    pb = synth.generate(base["config"], **over)
    f = synth.fields(base["config"], x_rand=False, **over)
    ap = assemble(f["params"], f)
    torch.cuda.synchronize()
    _compare(pb, ap)
    np.testing.assert_allclose(_host(ap.fs)[:2 * pb.Nc].reshape(-1, 2), pb.fs, rtol=1e-13, atol=0)
    np.testing.assert_allclose(ap.scales, pb.scales, rtol=1e-14)


def test_slab_assembly_with_global_row_maxima(dev):
    """P = 2 z-slabs: each rank assembles its owned rows (global column ids); with the maxima over both ranks the
    slabs are the row slices of the global Jacobian (synth.local_problem)."""
    from paper_1812_05540_b200 import assemble
    kw = dict(nx=12, ny=10, nz=64, recipe=2, perm_sigma=2.0)
    pb = synth.generate(**kw)
    f = synth.fields(x_rand=False, **kw)
    # first pass: every rank's own maxima; the "allreduce" is the max over the two passes
    maxima = [assemble(f["params"], f, rank=r, nranks=2, global_max=lambda m: m).row_max for r in range(2)]
    gmax = np.max(np.array(maxima), axis=0)
    for r in range(2):
        ap = assemble(f["params"], f, rank=r, nranks=2, global_max=lambda m: gmax)
        lp = synth.local_problem(pb, r, 2)
        rows = {"uu": (lp.node0, lp.Nn), "uf": (lp.node0, lp.Nn), "fu": (lp.cell0, lp.Nc), "ff": (lp.cell0, lp.Nc)}
        _compare(pb, ap, rows)
        np.testing.assert_allclose(_host(ap.fs)[:2 * lp.Nc].reshape(-1, 2), pb.fs[lp.cell0:lp.cell0 + lp.Nc], rtol=1e-13)


def test_solve_on_the_device_assembled_jacobian(dev):
    """Fields -> tsp_assemble -> tsp_create(inputs on the device) -> b = A x_rand on the device -> FGMRES: the same
    iteration count as the host-generated problem and the same solution to the solver tolerance."""
    from paper_1812_05540_b200 import Tsp, assemble
    pb = synth.generate("C2")
    f = synth.fields("C2")
    ap = assemble(f["params"], f)
    g = Tsp(ap, device_inputs=True).setup()
    xr = torch.from_numpy(f["x_rand"]).to(dev)
    b = torch.empty_like(xr)
    g.apply_operator(xr, b)
    torch.cuda.synchronize()
    assert np.linalg.norm(_host(b) - pb.b) <= 1e-12 * np.linalg.norm(pb.b)
    x = torch.zeros_like(xr)
    info = g.solve(b, x, rtol=1e-8)
    h = Tsp(pb).setup()
    xh = torch.zeros_like(xr)
    ih = h.solve(torch.from_numpy(pb.b).to(dev), xh, rtol=1e-8)
    assert info["status"] == "OK" and abs(info["iterations"] - ih["iterations"]) <= 1
    assert torch.linalg.norm(x - xh) <= 1e-6 * torch.linalg.norm(xh)
    g.close(); h.close()


def test_slab_pipeline_from_fields_is_rank_invariant(dev):
    """The multi-GPU bench pipeline on the in-process communicator: every rank assembles its slab from the global
    fields (row maxima combined over the ranks), creates its handle from device blocks, forms b = A x_rand on the
    device (a collective operator) and solves -- the glued solution and the iteration count equal the single-rank
    run of the same pipeline BITWISE."""
    import threading
    from paper_1812_05540_b200 import LocalWorld, Tsp, TSP_COMM_LOCAL, assemble
    kw = dict(nx=12, ny=10, nz=64, recipe=2, perm_sigma=2.0)
    f = synth.fields(**kw)
    prm = f["params"]
    s = synth.sizes(prm["nx"], prm["ny"], prm["nz"])

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
                    ap = assemble(prm, f, rank=r, nranks=P, stream=st, global_max=gmax(r))
                    _, _, n0, nn, c0, ncl = synth.slab_partition(prm["nx"], prm["ny"], prm["nz"], 16, r, P)
                    xr = f["x_rand"]
                    xl = np.concatenate([xr[3 * n0:3 * (n0 + nn)], xr[3 * s["Nn"] + 2 * c0:3 * s["Nn"] + 2 * (c0 + ncl)]])
                    kwc = dict(rank=r, nranks=P, comm_kind=TSP_COMM_LOCAL, comm_arg=world.h) if P > 1 else {}
                    g = Tsp(ap, stream=st, **kwc).setup()
                    b = torch.empty(ap.n, dtype=torch.float64, device=dev)
                    g.apply_operator(_cuda_t(xl), b)
                    x = torch.zeros_like(b)
                    info = g.solve(b, x, rtol=1e-8)
                    torch.cuda.synchronize()
                    out[r] = (x.cpu().numpy(), info["iterations"], nn)
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

    (x1, it1, _), = run(1)
    parts = run(2)
    u = np.concatenate([p[0][:3 * p[2]] for p in parts])
    fl = np.concatenate([p[0][3 * p[2]:] for p in parts])
    assert np.array_equal(np.concatenate([u, fl]), x1)
    assert parts[0][1] == parts[1][1] == it1


def _cuda_t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()
