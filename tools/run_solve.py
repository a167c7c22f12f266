"""Developer driver: one setup + one solve on a config (for ncu / sanitizer runs)."""
import argparse, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_1812_05540_b200 import Tsp
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4"); ap.add_argument("--maxit", type=int, default=20)
ap.add_argument("--applies", type=int, default=0)
a = ap.parse_args()
pb = synth.generate(a.config)
g = Tsp(pb).setup()
b = torch.from_numpy(pb.b).cuda(); x = torch.zeros(pb.n, dtype=torch.float64, device="cuda")
for _ in range(a.applies):
    g.apply_preconditioner(b, x)
if a.maxit:
    info = g.solve(b, x, max_iters=a.maxit)
    print(info)
torch.cuda.synchronize()
