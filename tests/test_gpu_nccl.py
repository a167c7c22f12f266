"""Row (e) over the real NCCL transport: two processes, one GPU each (cuda:0, cuda:1), the communicator bootstrapped
exactly as bench.py does it (tsp_nccl_unique_id on rank 0, broadcast through torch.distributed).  The assertion is
the design invariant: the sharded operator, one Algorithm 1 application and the FGMRES solution
are BITWISE identical to the single-GPU run, for both AMG layouts (distributed and replicated coarse levels) and
the Chebyshev smoother.  Skipped when fewer than two GPUs are visible (the in-process communicator of
tests/test_gpu_multirank.py covers the same schedule on one GPU)."""
import os
import socket

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GRID = dict(nx=12, ny=10, nz=64, recipe=2, perm_sigma=2.0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(pb, v, rank, ws, opts):
    from paper_1812_05540_b200 import TSP_COMM_NCCL, Tsp, nccl_unique_id
    import torch.distributed as dist
    kw = {}
    src, vv, bb = pb, v, pb.b
    if ws > 1:
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        kw = dict(rank=rank, nranks=ws, comm_kind=TSP_COMM_NCCL, comm_arg=obj[0])
        src = synth.local_problem(pb, rank, ws)
        vv, bb = src.local(v, pb.Nn), src.local(pb.b, pb.Nn)
    g = Tsp(src, **kw, **opts).setup()
    dv = torch.from_numpy(np.ascontiguousarray(vv)).cuda()
    z, y = torch.empty_like(dv), torch.empty_like(dv)
    g.apply_preconditioner(dv, z)
    g.apply_operator(dv, y)
    x = torch.zeros_like(dv)
    info = g.solve(torch.from_numpy(np.ascontiguousarray(bb)).cuda(), x, rtol=1e-8)
    torch.cuda.synchronize()
    out = dict(z=z.cpu().numpy(), y=y.cpu().numpy(), x=x.cpu().numpy(), it=info["iterations"])
    g.close()
    return out


def _worker(rank, ws, port, opts, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        pb = synth.generate(**GRID)
        v = np.random.default_rng(21).uniform(-1, 1, pb.n)
        out = _run(pb, v, rank, ws, opts)
        q.put((rank, out, None))
    except Exception as e:   # pragma: no cover - surfaced in the parent
        q.put((rank, None, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("opts", [dict(replicate_rows=32768), dict(replicate_rows=64), dict(amg_smoother=2)])
def test_nccl_two_gpus_bitwise_equals_one(opts):
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs (the in-process communicator covers the schedule on one)")
    import torch.multiprocessing as mp
    pb = synth.generate(**GRID)
    v = np.random.default_rng(21).uniform(-1, 1, pb.n)
    one = _run(pb, v, 0, 1, opts)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, opts, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(2):
        r, out, err = q.get(timeout=600)
        assert err is None, err
        res[r] = out
    for p in ps:
        p.join(timeout=60)
    lps = [synth.local_problem(pb, r, 2) for r in range(2)]
    for key in ("y", "z", "x"):
        u = np.concatenate([res[r][key][:3 * lps[r].Nn] for r in range(2)])
        f = np.concatenate([res[r][key][3 * lps[r].Nn:] for r in range(2)])
        assert np.array_equal(np.concatenate([u, f]), one[key]), key
    assert res[0]["it"] == res[1]["it"] == one["it"]
