"""Staircase benchmark (NEXT-f4 i): FGMRES iterations and times on the four Table 2 grids, rtol 1e-8 and 1e-6."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_1812_05540_b200 import Tsp
# STAIR_OPTS=amg_smoother=1,second_stage=1,local_sweeps=3 : the paper's staircase settings
opts = {k: int(v) for k, v in (kv.split("=") for kv in filter(None, os.environ.get("STAIR_OPTS", "").split(",")))}
print("options:", opts or "defaults", flush=True)
for lvl in ("ST0", "ST1", "ST2", "ST3"):
    pb = synth.generate(lvl)
    g = Tsp(pb, **opts)
    torch.cuda.synchronize(); t = time.time(); g.setup(); torch.cuda.synchronize(); ts = time.time() - t
    b = torch.from_numpy(pb.b).cuda()
    for rtol in (1e-8, 1e-6):
        x = torch.zeros(pb.n, dtype=torch.float64, device="cuda")
        info = g.solve(b, x, rtol=rtol, max_iters=1000)
        print(f"{lvl} {pb.nx}x{pb.ny}x{pb.nz} dof {pb.n} rtol {rtol:.0e}: {info['iterations']} it ({info['status']}), "
              f"solve {info['t_solve_s']*1e3:.1f} ms, setup {ts*1e3:.1f} ms", flush=True)
    g.close()
