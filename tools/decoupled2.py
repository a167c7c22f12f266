import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_1812_05540_b200 import Tsp
cfg = sys.argv[1]
pb = synth.generate(cfg)
nu = 3 * pb.Nn
flow = len(sys.argv) > 2 and sys.argv[2] == "flow"
if flow:
    pb.uf_val[:] = 0.0; pb.fu_val[:] = 0.0
    b = pb.b.copy(); b[:nu] = 0.0
else:
    b = pb.b
g = Tsp(pb).setup()
x = torch.zeros(pb.n, dtype=torch.float64, device="cuda")
info = g.solve(torch.from_numpy(b).cuda(), x, max_iters=1500)
print(cfg, "flow-only" if flow else "coupled", os.environ.get("TSP_DEV_PCYC", 1), os.environ.get("TSP_DEV_MCYC", 1), os.environ.get("TSP_DEV_ISW", 1), info["iterations"], info["status"], "%.1f ms/it" % (info["t_solve_s"] * 1e3 / max(info["iterations"], 1)))
