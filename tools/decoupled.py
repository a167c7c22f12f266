"""Developer: FGMRES iterations of the decoupled mechanics-only / flow-only problems (A_uf = A_fu = 0) vs coupled."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_1812_05540_b200 import Tsp
cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
pb = synth.generate(cfg)
nu = 3 * pb.Nn
def run(pb, b, **o):
    g = Tsp(pb, **o).setup()
    x = torch.zeros(pb.n, dtype=torch.float64, device="cuda")
    info = g.solve(torch.from_numpy(b).cuda(), x, max_iters=1500)
    g.close()
    return info["iterations"], info["status"]
print(cfg, "coupled", run(pb, pb.b))
pb.uf_val[:] = 0.0; pb.fu_val[:] = 0.0
bu = pb.b.copy(); bu[nu:] = 0.0
bf = pb.b.copy(); bf[:nu] = 0.0
print(cfg, "mechanics only", run(pb, bu))
print(cfg, "flow only", run(pb, bf))
