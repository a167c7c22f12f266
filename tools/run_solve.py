"""Developer driver: one setup + one solve on a config (for ncu / sanitizer runs).
--prof prints the live per-kernel-class breakdown (CUDA events on the solver stream)."""
import argparse, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_1812_05540_b200 import Tsp
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4"); ap.add_argument("--maxit", type=int, default=20)
ap.add_argument("--applies", type=int, default=0)
ap.add_argument("--prof", action="store_true")
a = ap.parse_args()
pb = synth.generate(a.config)
g = Tsp(pb).setup()
b = torch.from_numpy(pb.b).cuda(); x = torch.zeros(pb.n, dtype=torch.float64, device="cuda")
for _ in range(a.applies):
    g.apply_preconditioner(b, x)
if a.maxit:
    if a.prof:
        g.solve(b, x, max_iters=3)
        g.prof_enable(True)
    info = g.solve(b, x, max_iters=a.maxit)
    print(info)
    if a.prof:
        p = g.prof_read()
        tot = sum(v["ms"] for v in p.values())
        for k, v in sorted(p.items(), key=lambda kv: -kv[1]["ms"]):
            print(f"{k:14s} {v['launches']:7d} {v['ms']:9.2f} ms {100*v['ms']/tot:5.1f}%  "
                  f"{v['bytes']/max(v['ms'],1e-9)/1e6:7.0f} GB/s  {v['ms']/v['launches']*1e3:8.1f} us/launch")
torch.cuda.synchronize()
