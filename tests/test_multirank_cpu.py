"""Host-side logic of the z-slab decomposition (row e) on CPU with world_size 2
over gloo: every rank slices its owned rows from the seeded global problem, the
slices tile the global matrices exactly, the partition matches the library's
tsp_partition, and the NCCL id broadcast path carries 128 bytes unchanged.  The
device path itself is covered bitwise by tests/test_gpu_multirank.py."""
import os
import socket

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, grid, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        pb = synth.generate(**grid)
        lp = synth.local_problem(pb, rank, ws)
        # 1) the partition agrees with the C-ABI library (host function, no GPU needed)
        from paper_1812_05540_b200 import partition
        assert tuple(partition(pb.nx, pb.ny, pb.nz, 16, rank, ws)) == synth.slab_partition(pb.nx, pb.ny, pb.nz, 16, rank, ws)
        # 2) the id broadcast path used by bench.py
        obj = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        assert obj[0] == bytes(range(128))
        # 3) gather every rank's slice on rank 0
        mine = {k: getattr(lp, k) for k in ("uu_rowptr", "uu_col", "uu_val", "uf_rowptr", "uf_col", "uf_val",
                                            "fu_rowptr", "fu_col", "fu_val", "ff_rowptr", "ff_col", "ff_val", "fs")}
        mine.update(Nn=lp.Nn, Nc=lp.Nc, node0=lp.node0, cell0=lp.cell0,
                    b=lp.local(pb.b, pb.Nn))
        parts = [None] * ws
        dist.all_gather_object(parts, mine)
        if rank == 0:
            ok = []
            assert sum(p["Nn"] for p in parts) == pb.Nn and sum(p["Nc"] for p in parts) == pb.Nc
            for name in ("uu", "uf", "fu", "ff"):
                rp = np.concatenate([[0]] + [np.diff(p[name + "_rowptr"]) for p in parts]).cumsum()
                ok.append(np.array_equal(rp, getattr(pb, name + "_rowptr")))
                ok.append(np.array_equal(np.concatenate([p[name + "_col"] for p in parts]), getattr(pb, name + "_col")))
                ok.append(np.array_equal(np.concatenate([p[name + "_val"] for p in parts]), getattr(pb, name + "_val")))
            ok.append(np.array_equal(np.concatenate([p["fs"] for p in parts]), pb.fs))
            u = np.concatenate([p["b"][:3 * p["Nn"]] for p in parts])
            f = np.concatenate([p["b"][3 * p["Nn"]:] for p in parts])
            ok.append(np.array_equal(np.concatenate([u, f]), pb.b))
            # slabs are whole z-blocks: the first owned plane of every rank is a multiple of 16
            ok.append(all(p["cell0"] % (16 * pb.nx * pb.ny) == 0 for p in parts))
            q.put(all(ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ws", [2, 3])
def test_slab_slices_tile_the_problem(ws):
    grid = dict(nx=6, ny=5, nz=48, recipe=2, perm_sigma=2.0)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_worker, args=(ws, _free_port(), grid, q), nprocs=ws, join=True, start_method="spawn")
    assert q.get(timeout=60)
